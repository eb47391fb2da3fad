// rows_tma.cuh -- TMA-staged row sweeps (sweep 1 and sweep 3) for L >= 64.
//
// Same algebra as k_sweep1 / k_sweep3 (reference solvers.py:300-321 and
// :395-432), different data movement, the B200 way:
//   * a persistent CTA walks its lines (c, row) with stride gridDim.x;
//   * the full rows a line needs (sweep 1: the state row X0; sweep 3: the
//     y-inverted work row A, plus X0 for basic-type schemes) and the phase
//     row chi are fetched with cp.async.bulk (TMA bulk copy) into a ring of
//     NSTAGE shared-memory stages completed on mbarriers, NSTAGE-1 lines
//     ahead -- loads in flight hold no registers and no warps;
//   * the stage's main row doubles as the FFT exchange buffer once every
//     thread has read its inputs (padded layout, bank-conflict free);
//   * S/T slots (phase 1 only) are read straight from global memory after an
//     L2 bulk prefetch of the row's phase-1 extent one line ahead.
#pragma once
#include "sweeps.cuh"

namespace fftc {

#ifndef FFTC_ST_NSTAGE
#define FFTC_ST_NSTAGE 1
#endif

// resident CTAs per SM the 8-per-thread rows of 512 size their registers for
// (sweep 1: 64 threads per channel; sweep 3: 64 threads per CTA)
#ifndef FFTC_ROW512_MINB1
#define FFTC_ROW512_MINB1 4
#endif
#ifndef FFTC_ROW512_MINB3
#define FFTC_ROW512_MINB3 6
#endif
// em_sub sweep 1 on 8-per-thread rows: both channels (Rq, Jq) in one thread
// (1), or split over two thread groups with a shared-memory handoff (0)
#ifndef FFTC_ROW512_CPT2
#define FFTC_ROW512_CPT2 1
#endif
#ifndef FFTC_ROW512_MINBC
#define FFTC_ROW512_MINBC 6
#endif
// The same for em (16-per-thread rows, 32 values per thread).  Measured, split
// groups -> one thread (us): em at 2048^2 115.6 -> 111.5, at 512^3 4602 ->
// 3789, but at 1024^2 35.3 -> 37.0, so rows of 1024 keep the split; em_sub on
// 16-per-thread rows loses (2048^2 134.3 -> 142.5, 1024^2 38.9 -> 43.0: its
// prologue needs the registers) and keeps the split there.
#ifndef FFTC_ROW_CPT2_EM
#define FFTC_ROW_CPT2_EM 1
#endif
#ifndef FFTC_ROW_CPT2_MINB16
#define FFTC_ROW_CPT2_MINB16 2
#endif
// Variant V of the em_sub row sweeps for the memory-lean schedule (abi.cu,
// compact S/T slots, one work field): 0 = the normal sweeps; 1 = sweep 1 of
// the flux channel Jq alone; 2 = sweep 1 of the residual field Rq alone;
// 3 = sweep 3 over compact slots.  V > 0 stages rank codes (chiR, 2 bytes per
// voxel) instead of phase flags.
template <int S, int SW, int L, int V = 0>
struct RowTma {
  static constexpr int E = row_e(L, S);  // 16, or 8 on rows of 512 of the substituted schemes (sweeps.cuh)
  static constexpr int T = L / E;
  static constexpr bool LEAN = V != 0;
  // channels carried by one thread: em_sub's two sweep-1 channels on
  // 8-per-thread rows (16 values per thread, as one channel of 16): the
  // prologue runs once per element with no handoff between thread groups,
  // and one set of twiddle powers serves both transforms
  static constexpr int CPT = (SW == 1 && !LEAN &&
                              ((S == EM_SUB && E == 8 && FFTC_ROW512_CPT2) || (S == EM && L != 1024 && FFTC_ROW_CPT2_EM)))
                                 ? 2
                                 : 1;
  static constexpr int CH = (SW == 1 && !LEAN && CPT == 1) ? Sweep1Traits<S>::C : 1;
  static constexpr int THREADS = CH * T;
  static constexpr bool X0_ROW = (SW == 3) && (S == BASIC || S == BASIC_SUB);  // extra staged row
  // sweep 1 of the substituted schemes also stages its S (and T) rows over
  // the phase-1 extent; those areas are LP long so the first one can serve
  // as channel 1's exchange buffer once the inputs are in registers
  static constexpr int ST_ROWS = (SW == 1 && S == BASIC_SUB) ? 1 : 0;
  static constexpr int LP = Plan<L, E>::LP;
  static constexpr int ST_OFF = LP + (X0_ROW ? L : 0);
  static constexpr int CHI_OFF = ST_OFF + ST_ROWS * LP;     // double2 units
  static constexpr int CHI_BYTES = LEAN ? 2 * L : L;        // phase flags (or rank codes) of the row
  static constexpr int STAGE = CHI_OFF + CHI_BYTES / 16;
  // twiddle table copied to shared memory (swizzled, L/2 entries) instead of
  // read through L1 (~39 KB left beside the stages), paid for with a
  // single-stage ring; measured at 2048^2 (us): sweep 1 em 116.5 -> 114.8,
  // em_sub 136.0 -> 135.0, basic 73.2 -> 69.5 (1024^3: 20.6 -> 18.5 ms); sweep 3 basic 85.8 -> 79.7, basic_sub 114.5 ->
  // 94.7, em_sub 97.0 -> 93.3, but em 56.6 -> 61.7 (the lightest sweep loses
  // more from the shallower ring than it gains), so em's sweep 3 keeps two
  // stages.  FFTC_ROW_SMEMTW=0 switches it off.
#ifndef FFTC_ROW_SMEMTW
#define FFTC_ROW_SMEMTW 1
#endif
  // (at 1024 em_sub's sweep 3 measured 34.4 -> 36.3 us with it: 2048 and up)
  // (basic_sub's sweep 1 already stages its S row in a single stage; the table
  // on top measured 80.2 -> 87.8 us, so it keeps the L1 path)
#ifndef FFTC_TWS_MINL
#define FFTC_TWS_MINL 1024
#endif
  static constexpr bool TWS = FFTC_ROW_SMEMTW && L >= FFTC_TWS_MINL &&
                              ((SW == 1 && ST_ROWS == 0) ||
                               (SW == 3 && (S == BASIC || S == BASIC_SUB)) || (SW == 3 && S == EM_SUB && L >= 2048));
  static constexpr int NSTAGE = TWS ? 1 : (ST_ROWS ? FFTC_ST_NSTAGE : 2);
  static constexpr int XBUF = ((CH == 2 || CPT == 2) && ST_ROWS == 0) ? LP : 0;  // exchange buffer of channel 1
  static constexpr int TWOFF = NSTAGE * STAGE + XBUF;              // double2 units
  static constexpr int SMEM = (TWOFF + (TWS ? L / 2 : 0)) * (int)sizeof(double2);
  static constexpr unsigned TX = (unsigned)(L * sizeof(double2) * (1 + (X0_ROW ? 1 : 0)) + CHI_BYTES);
  // resident CTAs per SM the register budget is sized for: the tuned values
  // for sweep 3 and at L != 1024; sweep-1 rows of 1024 (64 threads per
  // channel) fill the SM up to 16 warps or the shared-memory limit, whichever
  // comes first (1024^2 em_sub sweep 1 44.3 -> 41.0 us; the same rule cost
  // em sweep 3 at 1024 23.2 -> 24.3 us and em_sub sweep 1 at 512^3 5.37 ->
  // 5.78 ms, so those keep the tuned values)
  static constexpr int MINB_TUNED = SW == 3 ? 3 : (ST_ROWS ? 1 : 2);
  static constexpr int MINB_FILL = (232448 / (SMEM + 1024)) < (512 / THREADS) ? (232448 / (SMEM + 1024)) : (512 / THREADS);
  static constexpr int MINB_E8 =
      SW == 3 ? FFTC_ROW512_MINB3 : (CPT == 2 ? FFTC_ROW512_MINBC : (CH == 2 ? FFTC_ROW512_MINB1 : 2 * FFTC_ROW512_MINB1));
  static constexpr int MINB = E == 8 ? MINB_E8
                                     : (CPT == 2 ? FFTC_ROW_CPT2_MINB16
                                                 : ((L != 1024 || SW == 3) ? MINB_TUNED : (MINB_FILL > 1 ? MINB_FILL : 1)));
};

template <int S, int SW, int L, int V = 0>
__device__ __forceinline__ void rows_tma_issue(const Args& a, double2* stage, uint64_t* bar, long long line,
                                               long long rows) {
  using K = RowTma<S, SW, L, V>;
  const int c = (int)(line / rows);
  const long long row = line - (long long)c * rows;
  const size_t off = (size_t)c * a.N + (size_t)row * L;
  unsigned tx = K::TX;
  int x0 = 0;
  unsigned nb = 0;
  if constexpr (K::ST_ROWS > 0) {
    const int2 ext = a.row_ext[row];
    if (ext.x < ext.y) {
      x0 = ext.x & ~1;
      nb = (unsigned)((ext.y - x0) * sizeof(double2) + 15) & ~15u;
      tx += K::ST_ROWS * nb;
    }
  }
  mbar_expect_tx(bar, tx);
  bulk_g2s(stage, SW == 1 ? a.X[0] + off : a.A + work_off(a, c, row), (unsigned)(L * sizeof(double2)), bar);
  if constexpr (K::X0_ROW) bulk_g2s(stage + K::LP, a.X[0] + off, (unsigned)(L * sizeof(double2)), bar);
  if constexpr (K::ST_ROWS > 0) {
    if (nb) {
      bulk_g2s(stage + K::ST_OFF + x0, a.X[1] + off + x0, nb, bar);
      if constexpr (K::ST_ROWS > 1) bulk_g2s(stage + K::ST_OFF + K::LP + x0, a.X[2] + off + x0, nb, bar);
    }
  }
  if constexpr (K::LEAN)
    bulk_g2s(stage + K::CHI_OFF, a.chiR + (size_t)row * L, (unsigned)K::CHI_BYTES, bar);  // rank codes
  else
    bulk_g2s(stage + K::CHI_OFF, a.chiT + (size_t)row * L, (unsigned)L, bar);  // thread-blocked chi row
}

// a thread's E phase flags (chiT row bytes t*E .. t*E+E-1, element i = byte i)
template <int E>
struct ChiBytes {
  uint32_t w[E / 4];
  __device__ __forceinline__ bool in1(int i) const { return ((w[i >> 2] >> ((i & 3) << 3)) & 0xffu) != 0u; }
};
template <int E>
__device__ __forceinline__ ChiBytes<E> load_chi(const uint8_t* chi_s, int t) {
  static_assert(E == 8 || E == 16, "thread-blocked chi rows hold 8 or 16 flags per thread");
  ChiBytes<E> r;
  if constexpr (E == 16) {
    const uint4 c = *reinterpret_cast<const uint4*>(chi_s + 16 * t);
    r.w[0] = c.x; r.w[1] = c.y; r.w[2] = c.z; r.w[3] = c.w;
  } else {
    const uint2 c = *reinterpret_cast<const uint2*>(chi_s + 8 * t);
    r.w[0] = c.x; r.w[1] = c.y;
  }
  return r;
}

// a thread's E rank codes of the compact layout (chiR row entries t*E ..
// t*E+E-1): element i is phase 1 when its code is nonzero, and its S/T slot
// is the row's compact base + code - 1
template <int E>
struct ChiCodes {
  uint32_t w[E / 2];
  __device__ __forceinline__ int code(int i) const { return (int)((w[i >> 1] >> ((i & 1) << 4)) & 0xffffu); }
  __device__ __forceinline__ bool in1(int i) const { return code(i) != 0; }
};
template <int E>
__device__ __forceinline__ ChiCodes<E> load_codes(const uint8_t* chi_s, int t) {
  ChiCodes<E> r;
  const uint4 c0 = *reinterpret_cast<const uint4*>(chi_s + 2 * E * t);
  r.w[0] = c0.x; r.w[1] = c0.y; r.w[2] = c0.z; r.w[3] = c0.w;
  if constexpr (E == 16) {
    const uint4 c1 = *reinterpret_cast<const uint4*>(chi_s + 32 * t + 16);
    r.w[4] = c1.x; r.w[5] = c1.y; r.w[6] = c1.z; r.w[7] = c1.w;
  }
  return r;
}
template <bool LEAN, int E>
struct PhaseRow;
template <int E>
struct PhaseRow<false, E> {
  using type = ChiBytes<E>;
  static __device__ __forceinline__ type load(const uint8_t* chi_s, int t) { return load_chi<E>(chi_s, t); }
};
template <int E>
struct PhaseRow<true, E> {
  using type = ChiCodes<E>;
  static __device__ __forceinline__ type load(const uint8_t* chi_s, int t) { return load_codes<E>(chi_s, t); }
};
// S/T slot of element i of this thread: full-grid (off + x) or compact (base + code - 1)
template <int E>
__device__ __forceinline__ size_t st_slot(const ChiBytes<E>&, int, size_t off, int x) { return off + x; }
template <int E>
__device__ __forceinline__ size_t st_slot(const ChiCodes<E>& cc, int i, size_t base, int) {
  return base + (size_t)(cc.code(i) - 1);
}

template <int S, int SW, int L, int V = 0>
constexpr bool rows_prefetch_slots() {
  return (S == BASIC_SUB || S == EM_SUB) && RowTma<S, SW, L, V>::ST_ROWS == 0;
}

// L2 prefetch of the phase-1 extent of the S/T (and em_sub sweep-3 Q) rows;
// `ext` (that line's row_ext entry) was loaded one line earlier so the
// prefetching warp never waits on it in front of the block barrier
template <int S, int SW, int L, int V = 0>
__device__ __forceinline__ void rows_tma_prefetch_slots(const Args& a, int line, int lines, int rows, int2 ext) {
  if (!rows_prefetch_slots<S, SW, L, V>() || line >= lines) return;
  const int c = line / rows;
  const int row = line - c * rows;
  if (ext.x >= ext.y) return;
  const size_t off = (size_t)c * a.N + (size_t)row * L + (ext.x & ~1);
  const unsigned nb = (unsigned)((ext.y - (ext.x & ~1)) * sizeof(double2) + 15) & ~15u;
  if (SW == 3 && S == EM_SUB) l2_prefetch(a.X[0] + off, nb);
  if constexpr (V != 0) {  // compact slots: the row's phase-1 run is contiguous
    const long long b = a.rowoff[row], e = a.rowoff[row + 1];
    const size_t coff = (size_t)c * a.M + (size_t)b;
    const unsigned cb = (unsigned)((e - b) * (long long)sizeof(double2));
    l2_prefetch(a.X[1] + coff, cb);
    l2_prefetch(a.X[2] + coff, cb);
  } else {
    l2_prefetch(a.X[1] + off, nb);
    if (S == EM_SUB) l2_prefetch(a.X[2] + off, nb);
  }
}

// em_sub sweep 1 with its two channels (Rq: channel 0, Jq: channel 1): thread
// (ch, t) evaluates the prologue (solvers.py:398-420: A applied to (Q, S, T),
// the pinned flux) of elements H*E/2 .. H*E/2 + E/2 - 1 for BOTH channels, so
// apply_A and the S/T loads run once per element instead of once per channel,
// keeps its own channel's values and stages the partner's (thread (1-ch, t))
// at the element's position in `other` (channel 0's main row / channel 1's
// exchange buffer; each position is read and rewritten by one thread only).
template <int H, int L, int E, int NQ>
__device__ __forceinline__ void em_sub_prologue_half(const Args& a, double2 (&v)[1][E], const double2* st,
                                                     const ChiBytes<E>& cb, double2* other, int t, int c, size_t off,
                                                     double2 dl, double (&acc)[NQ]) {
  // S/T loads (phase 1 only, L2-prefetched) in batches of NB issued ahead of
  // the batch's staging stores; interleaved with them each would wait one latency
  constexpr int NB = 4;
#pragma unroll
  for (int k0 = 0; k0 < E / 2; k0 += NB) {
    double2 sv[NB], tv[NB];
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      const int x = pos_first<L, E>(false, t, H * (E / 2) + k0 + u);
      sv[u] = tv[u] = czero();
      if (cb.in1(H * (E / 2) + k0 + u)) {
        sv[u] = a.X[1][off + x];
        tv[u] = a.X[2][off + x];
      }
    }
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      const int i = H * (E / 2) + k0 + u;
      const int x = pos_first<L, E>(false, t, i);
      const bool in1 = cb.in1(i);
      const double2 q = st[x];
      const AugFlux f = apply_A(a, in1, q, sv[u], tv[u]);
      double2 jq, js;
      pinned_flux(a, in1, f.jq, f.js, dl, jq, js);
      acc_c<NQ>(acc, c, jq);
      if (in1) acc[NQ - 1] += cabs2(js);
      const double2 rq = csub(f.jq, cmul(a.s0, q));
      v[0][i] = H == 0 ? rq : jq;
      other[x] = H == 0 ? jq : rq;
    }
  }
}

template <int S, int SW, int L, int V = 0>
__global__ void __launch_bounds__(RowTma<S, SW, L, V>::THREADS, RowTma<S, SW, L, V>::MINB) k_rows_tma(Args a) {
  using K = RowTma<S, SW, L, V>;
  static_assert(V == 0 || S == EM_SUB, "the compact variants are em_sub sweeps");
  static_assert(V == 0 || (SW == 1) == (V != 3), "variants 1, 2 are sweep 1; variant 3 is sweep 3");
  constexpr int E = K::E, T = K::T, CH = K::CH;
  constexpr int NQ = (SW == 1) ? (V == 2 ? 1 : Sweep1Traits<S>::NQ) : 6;
  constexpr bool INV = (SW == 3);
  extern __shared__ __align__(128) double2 smem[];
  __shared__ uint64_t bars[K::NSTAGE];
  __shared__ double2 sdelta[3];
  if (a.st->stopped) return;
  const int t = threadIdx.x % T, ch = threadIdx.x / T;
  const bool jchan = V == 1 ? true : (V == 2 ? false : (ch == CH - 1));
  // 32-bit line bookkeeping (axes <= 4096, so rows * d <= 3 * 2^24): keeps the
  // loop state in registers instead of local memory
  const int rows = a.ny * a.nz;
  const int lines = rows * a.d;
  const int nmine = (int)blockIdx.x < lines ? (lines - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < K::NSTAGE; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 3) sdelta[threadIdx.x] = a.st->delta[threadIdx.x];
  if constexpr (K::TWS)
    for (int i = threadIdx.x; i < L / 2; i += blockDim.x) smem[K::TWOFF + tw_swz(i)] = __ldg(&a.tw[0][i]);
  // phase-1 extent of the line after next, for the S/T prefetch
  const bool pf = rows_prefetch_slots<S, SW, L, V>() && threadIdx.x == blockDim.x - 1;
  int2 ext_next = make_int2(0, 0);
  if (pf && (int)blockIdx.x + (int)gridDim.x < lines) ext_next = a.row_ext[((int)blockIdx.x + (int)gridDim.x) % rows];
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = 0; s < K::NSTAGE && s < nmine; ++s)
      rows_tma_issue<S, SW, L, V>(a, smem + s * K::STAGE, &bars[s], blockIdx.x + (long long)s * gridDim.x, rows);
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  double2* xbuf = smem + K::NSTAGE * K::STAGE;
  double2* OUT = (SW == 1 && CH == 2 && ch == 1) ? a.B : a.A;
  for (int k = 0; k < nmine; ++k) {
    const int s = k % K::NSTAGE;
    const unsigned parity = (unsigned)((k / K::NSTAGE) & 1);
    const int line = (int)blockIdx.x + k * (int)gridDim.x;
    const int c = line / rows;
    const int row = line - c * rows;
    const size_t off = (size_t)c * a.N + (size_t)row * L;
    const double2 dl = sdelta[c];
    double2* st = smem + s * K::STAGE;
    const uint8_t* chi_s = reinterpret_cast<const uint8_t*>(st + K::CHI_OFF);
    if (pf) {
      const int2 ext = ext_next;
      const int l2 = line + 2 * (int)gridDim.x;
      if (l2 < lines) ext_next = a.row_ext[l2 % rows];
      rows_tma_prefetch_slots<S, SW, L, V>(a, line + (int)gridDim.x, lines, rows, ext);
    }
    mbar_wait(&bars[s], parity);
    const typename PhaseRow<K::LEAN, E>::type cb = PhaseRow<K::LEAN, E>::load(chi_s, t);
    // S/T slot base of this line: the full-grid row, or the row's compact run
    const size_t sbase = K::LEAN ? (size_t)c * a.M + (size_t)a.rowoff[row] : off;
    constexpr int CPT = K::CPT;
    double2 v[CPT][E];
    constexpr bool SPLIT = (SW == 1 && S == EM_SUB && CH == 2 && K::ST_ROWS == 0);
    if constexpr (CPT == 2) {
      // ---- prologue, both channels in this thread (solvers.py:303-311 /
      // :398-420): channel 0 = the residual field, channel 1 = the flux; the
      // S/T loads of a batch are issued before its arithmetic ----
      constexpr int NB = E == 8 ? 8 : 4;
#pragma unroll
      for (int b0 = 0; b0 < E; b0 += NB) {
        double2 sv[NB], tv[NB];
        if constexpr (S == EM_SUB) {
#pragma unroll
          for (int u = 0; u < NB; ++u) {
            sv[u] = tv[u] = czero();
            if (cb.in1(b0 + u)) {
              const int x = pos_first<L, E>(false, t, b0 + u);
              sv[u] = a.X[1][st_slot(cb, b0 + u, sbase, x)];
              tv[u] = a.X[2][st_slot(cb, b0 + u, sbase, x)];
            }
          }
        }
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          const int i = b0 + u;
          const int x = pos_first<L, E>(false, t, i);
          const bool in1 = cb.in1(i);
          const double2 q = st[x];
          if constexpr (S == EM_SUB) {
            const AugFlux f = apply_A(a, in1, q, sv[u], tv[u]);
            double2 jq, js;
            pinned_flux(a, in1, f.jq, f.js, dl, jq, js);
            acc_c<NQ>(acc, c, jq);
            if (in1) acc[NQ - 1] += cabs2(js);
            v[0][i] = csub(f.jq, cmul(a.s0, q));
            v[1][i] = jq;
          } else {  // EM
            const double2 j = cmul(sigma_at(a, in1), cadd(q, dl));
            acc_c<NQ>(acc, c, j);
            v[0][i] = cmul(in1 ? a.sm1 : a.sm2, q);
            v[1][i] = j;
          }
        }
      }
    } else if constexpr (SPLIT) {
      // ---- prologue, each element once (see em_sub_prologue_half) ----
      if (ch == 0) em_sub_prologue_half<0, L, E, NQ>(a, v, st, cb, xbuf, t, c, off, dl, acc);
      else em_sub_prologue_half<1, L, E, NQ>(a, v, st, cb, st, t, c, off, dl, acc);
    } else if constexpr (SW == 1) {
      // ---- prologue: fields to transform (solvers.py:303-311 / :398-420) ----
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int x = pos_first<L, E>(false, t, i);
        const bool in1 = cb.in1(i);
        const double2 q = st[x];
        if constexpr (S == BASIC) {
          const double2 j = cmul(sigma_at(a, in1), cadd(q, dl));
          v[0][i] = j;
          acc_c<NQ>(acc, c, j);
        } else if constexpr (S == EM) {
          if (jchan) {
            const double2 j = cmul(sigma_at(a, in1), cadd(q, dl));
            v[0][i] = j;
            acc_c<NQ>(acc, c, j);
          } else {
            v[0][i] = cmul(in1 ? a.sm1 : a.sm2, q);
          }
        } else {
          double2 sv = czero(), tv = czero();
          if (in1) {
            if constexpr (K::ST_ROWS >= 1) sv = st[K::ST_OFF + x];
            else sv = a.X[1][st_slot(cb, i, sbase, x)];
            if constexpr (S == EM_SUB) {
              if constexpr (K::ST_ROWS >= 2) tv = st[K::ST_OFF + K::LP + x];
              else tv = a.X[2][st_slot(cb, i, sbase, x)];
            }
          }
          const AugFlux f = apply_A(a, in1, q, sv, tv);
          if (jchan) {
            double2 jq, js;
            pinned_flux(a, in1, f.jq, f.js, dl, jq, js);
            v[0][i] = jq;
            acc_c<NQ>(acc, c, jq);
            if (in1) acc[NQ - 1] += cabs2(js);
          } else {
            v[0][i] = csub(f.jq, cmul(a.s0, q));
          }
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < E; ++i) v[0][i] = st[pos_first<L, E>(true, t, i)];
    }
    __syncthreads();  // the main row becomes exchange scratch
    double2* xb = (CH == 2 && ch == 1) ? (K::ST_ROWS ? st + K::ST_OFF : xbuf) : st;
    if constexpr (SPLIT) {
      // the partner's half of this channel, staged in this channel's buffer
      if (ch == 0) {
#pragma unroll
        for (int k = 0; k < E / 2; ++k) v[0][E / 2 + k] = st[pos_first<L, E>(false, t, E / 2 + k)];
      } else {
#pragma unroll
        for (int k = 0; k < E / 2; ++k) v[0][k] = xbuf[pos_first<L, E>(false, t, k)];
      }
      HalfSync{1 + ch, T}();  // every staged value is read before the first exchange overwrites it
    }
    if constexpr (CPT == 2) {
      // both channels through one transform (shared twiddle powers): channel 0
      // exchanges in the main row, channel 1 in xbuf
      const SmemBuf xb2{st, (int)(xbuf - st)};
      if constexpr (K::TWS) fft_line<L, E, 2, INV, false>(v, t, SmemTw{smem + K::TWOFF}, xb2, SyncAll{});
      else fft_line<L, E, 2, INV, false>(v, t, a.tw[0], xb2, SyncAll{});
    } else if constexpr (CH == 2) {
      // the two channels transform in separate buffers: each synchronises
      // only its own T threads (named barrier 1 + ch), not the whole CTA
      // (no barrier after the last exchange: the __syncthreads closing the
      // line comes before the buffer is written again)
      if constexpr (K::TWS)
        fft_line<L, E, 1, INV, false>(v, t, SmemTw{smem + K::TWOFF}, SmemBuf{xb, 0}, HalfSync{1 + ch, T});
      else
        fft_line<L, E, 1, INV, false>(v, t, a.tw[0], SmemBuf{xb, 0}, HalfSync{1 + ch, T});
    } else {
      if constexpr (K::TWS)
        fft_line<L, E, 1, INV, false>(v, t, SmemTw{smem + K::TWOFF}, SmemBuf{xb, 0}, SyncAll{});
      else
        fft_line<L, E, 1, INV, false>(v, t, a.tw[0], SmemBuf{xb, 0}, SyncAll{});
    }
    if constexpr (SW == 1) {
      const size_t woff = work_off(a, c, row);  // work field row (z-blocked in 3-D)
#pragma unroll
      for (int i = 0; i < E; ++i) OUT[woff + pos_last<L, E>(false, t, i)] = v[0][i];
      if constexpr (CPT == 2) {
#pragma unroll
        for (int i = 0; i < E; ++i) a.B[woff + pos_last<L, E>(false, t, i)] = v[1][i];
      }
    } else {
      // ---- epilogue: state update for iteration k+1 (solvers.py:303-308, :398-411) ----
      // Elements go in batches of NB: the batch's phase-1 state loads (L2-
      // prefetched) are all issued before its stores, so a thread waits for
      // the load latency E/NB times per line instead of once per element
      // (the stores may alias the loads, so the compiler cannot hoist them).
      constexpr int NB = 4;
#pragma unroll
      for (int b0 = 0; b0 < E; b0 += NB) {
        double2 qv[NB], sv[NB], tv[NB];
        bool in1v[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          const int x = pos_last<L, E>(true, t, b0 + u);
          in1v[u] = cb.in1(b0 + u);
          qv[u] = sv[u] = tv[u] = czero();
          if constexpr (S == BASIC_SUB) {
            if (in1v[u]) sv[u] = a.X[1][off + x];
          } else if constexpr (S == EM_SUB) {
            if (in1v[u]) {
              qv[u] = a.X[0][off + x];
              sv[u] = a.X[1][st_slot(cb, b0 + u, sbase, x)];
              tv[u] = a.X[2][st_slot(cb, b0 + u, sbase, x)];
            }
          }
        }
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          const int x = pos_last<L, E>(true, t, b0 + u);
          const bool in1 = in1v[u];
          const double2 gq = cscale(v[0][b0 + u], a.inv_n);
          double2 qn;
          if constexpr (S == BASIC) {
            qn = csub(cadd(st[K::LP + x], dl), cmul(gq, a.inv_s0));
            a.X[0][off + x] = qn;
          } else if constexpr (S == EM) {
            qn = cmul(cadd(a.two_s0_e0[c], gq), in1 ? a.inv_sum1 : a.inv_sum2);
            a.X[0][off + x] = qn;
          } else if constexpr (S == BASIC_SUB) {
            const double2 q = st[K::LP + x];
            qn = csub(cadd(q, dl), cmul(gq, a.inv_s0));
            a.X[0][off + x] = qn;
            if (in1) {
              const AugFlux f = apply_A(a, true, q, sv[u], czero());
              double2 jq, js;
              pinned_flux(a, true, f.jq, f.js, dl, jq, js);
              a.X[1][off + x] = csub(sv[u], cmul(js, a.inv_s0));
            }
          } else {
            const double2 wq = cadd(a.two_s0_e0[c], gq);
            double2 ws = czero(), wt = czero();
            if (in1) {
              const AugFlux f = apply_A(a, true, qv[u], sv[u], tv[u]);
              const double2 rs = csub(f.js, cmul(a.s0, sv[u]));
              ws = make_double2(-rs.x, -rs.y);
              wt = csub(f.jt, cmul(a.s0, tv[u]));
            }
            double2 sn, tn;
            em_sub_update(a, in1, wq, ws, wt, qn, sn, tn);
            a.X[0][off + x] = qn;
            if (in1) {
              a.X[1][st_slot(cb, b0 + u, sbase, x)] = sn;
              a.X[2][st_slot(cb, b0 + u, sbase, x)] = tn;
            }
          }
          acc_c<NQ>(acc, c, qn);
        }
      }
    }
    __syncthreads();  // stage s fully consumed (exchange, chi, X0 row)
    if (threadIdx.x == 0 && k + K::NSTAGE < nmine) {
      fence_proxy_async();
      rows_tma_issue<S, SW, L, V>(a, st, &bars[s], (long long)line + (long long)K::NSTAGE * gridDim.x, rows);
    }
  }
  double tot[NQ];
  if (grid_reduce<NQ>(acc, tot, a) && threadIdx.x == 0) {
    if constexpr (SW == 1) {
      if constexpr (V != 2) {  // (the residual-field sweep of the lean schedule carries no flux sums)
        for (int cc = 0; cc < a.d; ++cc)
          a.st->jmean[cc] = make_double2(tot[2 * cc] * a.inv_n, tot[2 * cc + 1] * a.inv_n);
        a.st->js2 = (NQ > 6) ? tot[NQ - 1] : 0.0;
      }
    } else {
      for (int cc = 0; cc < a.d; ++cc)
        a.st->delta[cc] = csub(a.e0[cc], make_double2(tot[2 * cc] * a.inv_n, tot[2 * cc + 1] * a.inv_n));
    }
  }
}

}  // namespace fftc
