// cols3_lg.cuh -- TMA-staged column passes of 3-D fields, line-group form
// (the y passes and the z pass with the Gamma projection, lines of 256..1024).
//
// Same algebra and the same tiles as round 1's k_col3_tma (spectral_ops.py:120-128
// in 3-D: a tile is W adjacent x-columns of all three components along the
// line axis, one cp.async.bulk.tensor per tile, two slots).  What changes is
// who synchronises with whom.  There a line's T threads were spread over all
// eight warps of its component (w fastest), so each of the four to eight FFT
// exchanges of a tile was a CTA-wide __syncthreads: all 24 warps moved in
// lockstep from an FP64-bound butterfly phase to a shared-memory-bound
// exchange phase and back, and neither pipe overlapped the other (ncu: FP64
// 28-45 %, barrier the top stall).  Here a line belongs to T consecutive
// threads (one, two or four warps), the FFT exchanges use a named barrier of
// that group only (__syncwarp at T = 32), and the twelve to twenty-four
// groups of a CTA drift apart: one group's exchange overlaps another's
// butterflies.  CTA-wide barriers remain where the tile's layout changes
// hands: inputs in registers, the projection's k.F^ exchange, outputs staged.
//
// The landing layout [c][pos][w] interleaves the W columns, so with t
// fastest a warp would read one column at a stride of 16 W bytes (W-way bank
// conflicts).  The tensor maps therefore carry the TMA swizzle whose span is
// one box row (32 / 64 / 128 B for W = 2 / 4 / 8): the 16-byte chunk index w
// of row pos becomes w ^ ((pos >> (3 - log2 W)) & (W - 1)), and eight
// consecutive line positions of one column fall in eight distinct 16-byte
// bank groups -- loads from the landing area and the staged outputs are
// conflict free.  Slots are 1024-byte aligned so the pattern is a function of
// the slot offset.
#pragma once
#include "cols3_tma.cuh"

namespace fftc {

#ifndef FFTC_COL3_GROUPSYNC
#define FFTC_COL3_GROUPSYNC 1  // 0: CTA-wide barriers in the transforms (A/B comparison)
#endif
// L2 prefetch of the tile after the one being loaded (1: on).  Measured
// slower at 512^3 (y forward 2.67 -> 2.84 ms, y inverse 2.22 -> 2.39 ms, z pass
// unchanged) and at 1024^3 (y forward 31 -> 39 ms): the prefetch's box rows
// queue on the same TMA unit as the loads and stores.
#ifndef FFTC_COL3_PF
#define FFTC_COL3_PF 0
#endif
// two-field passes (the EM-type z pass: field A transformed and stored, the
// flux field B Parseval-only) alternate A and B tiles (1) instead of all of A
// then all of B (0): A tiles then always use slot 0 and B tiles slot 1, so a B
// tile's load never waits for a store and A's store read-out overlaps B's work
#ifndef FFTC_COL3_ALT
#define FFTC_COL3_ALT 1
#endif

__device__ __forceinline__ void col3_prefetch(const CUtensorMap* tm, int x0, int2 oc) {
  asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(tm), "r"(2 * x0),
               "r"(0), "r"(oc.x), "r"(oc.y), "r"(0)
               : "memory");
}

// NCT components per tile (3: the projection pass needs them together; 1: the
// plain y passes may take them one at a time), WT columns per tile, NS slots
template <int L, int NCT = 3, int WT = col3_tile_w(L), int NS = 2>
struct Col3Lg {
  static constexpr int E = 8;
  static constexpr int T = L / E;  // threads of one line
  static constexpr int W = WT;     // columns per tile
  static constexpr int LGW = ilog2(W);
  static constexpr int NC = NCT;
  static constexpr int NL = NC * W;  // lines per tile
  static constexpr int THREADS = NL * T;
  static constexpr int LP = Plan<L, E>::LP;
  static constexpr int XS = LP;         // a line's own exchange buffer inside the slot
  static constexpr int SLOT = NL * XS;  // >= NL * L landing
  static constexpr int NSLOT = NS;
  // (+ 1024: the kernel aligns its slots inside the dynamic segment)
  static constexpr int SMEM = (NSLOT * SLOT + L / 2) * (int)sizeof(double2) + 1024;
  static constexpr unsigned TX = (unsigned)(NL * L * sizeof(double2));
  static_assert(W == 2 || W == 4 || W == 8, "swizzle spans of 32 / 64 / 128 bytes");
  static_assert(THREADS <= 1024 && T % 32 == 0, "block size; a line is whole warps");
  static_assert((SLOT * 16) % 1024 == 0, "slots keep the 1024-byte swizzle alignment");
  static_assert(NL <= 15 || T == 32, "one named barrier per line");
  static_assert(SMEM + 2048 <= 232448, "shared memory budget (with the kernel's static variables)");
  static_assert(NC == 3 || NC == 1, "whole vectors or single components");
  // entry of (component c, line position pos, column w) in the swizzled landing layout
  __device__ static __forceinline__ int land(int c, int pos, int w) {
    return ((c * L + pos) << LGW) | (w ^ ((pos >> (3 - LGW)) & (W - 1)));
  }
};

// Plain y passes on single-component tiles: 8 columns (128-byte box rows: half
// the TMA requests per byte of the 4-column vector tiles) and three slots, so
// the load of tile k+2, the transform of tile k and the store of tile k-1
// overlap.  Measured SLOWER where it ran (256^3: y forward 282 -> 314 us, y
// inverse 240 -> 270 us per field), so the vector tiles stay (FFTC_COL3_Y1 = 1
// builds it).
#ifndef FFTC_COL3_Y1
#define FFTC_COL3_Y1 0
#endif
// Lines of 1024: the vector tiles are two columns wide (32-byte box rows), and
// ncu shows the passes re-reading DRAM (1024^3: 70.1 GB read per launch
// against 51.5 GB algorithmic -- half-used 64-byte DRAM atoms whose other half
// is gone from L2 when the neighbouring tile asks for it).  Single-component
// tiles there are four columns wide (64-byte rows, three slots).
#ifndef FFTC_COL3_Y1_1024
#define FFTC_COL3_Y1_1024 1
#endif
template <int L>
struct Col3YSel {
  static constexpr bool Y1 = (FFTC_COL3_Y1 && L <= 512) || (FFTC_COL3_Y1_1024 && L == 1024);
  using type = Col3Lg<L, Y1 ? 1 : 3, Y1 ? (L == 1024 ? 4 : 8) : col3_tile_w(L), Y1 ? 3 : 2>;
};

// barrier over the T threads of one line
template <int T>
struct LineSync {
  int id;
  __device__ __forceinline__ void operator()() const {
#if FFTC_COL3_GROUPSYNC
    if constexpr (T == 32) __syncwarp();
    else asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(T) : "memory");
#else
    __syncthreads();
#endif
  }
};

// PEER: outputs go straight to their owning rank (PeerOut po) as bulk copies
// of whole tile rows -- the decomposed solve's transposes fused into the pass
// that produces the data (staged unswizzled: a bulk copy reads raw bytes).
template <int MODE, int L, bool PEER = false, class K = Col3Lg<L>>
__global__ void __launch_bounds__(K::THREADS, 1)
    k_col3_lg(Args a, Line3 g, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const PeerOut* __restrict__ po) {
  constexpr int E = K::E, T = K::T, W = K::W, NC = K::NC;
  constexpr bool MID = (MODE == MID_BASIC || MODE == MID_EM);
  constexpr bool INV_ONLY = (MODE == COL_INV);
  static_assert(!MID || NC == 3, "the projection needs whole vectors");
  extern __shared__ __align__(128) double2 smem_raw[];
  __shared__ uint64_t bars[K::NSLOT];
  if (!a.op_mode && a.st->stopped) return;
  // slots on 1024-byte boundaries of the shared window: the swizzle is a function of the slot offset
  double2* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u) / (unsigned)sizeof(double2);
  // (NC = 1: the tile's component comes with the tile, lcomp = 0 in the slot)
  const int t = threadIdx.x % T, line = threadIdx.x / T, w = line % W, lcomp = line / W;
  const int nstrips = a.nx / W;
  // Tiles of one field go round robin over the CTAs, field after field, so a
  // pass over field B alone (Line3::f0 = 1, the memory-lean schedule) deals a
  // CTA the same flux tiles in the same order as the two-field pass does.
  const int per_comp = g.nouter * nstrips;
  const int per_field = per_comp * (3 / NC);
  const int nper = (int)blockIdx.x < per_field ? (per_field - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  const int nmine = nper * g.nfields;
  auto coords = [&](int k, int& f, int& o, int& x0, int& c0) {
    // (nfields <= 2)
#if FFTC_COL3_ALT
    const int fl = g.nfields == 2 ? (k & 1) : 0;
    int r = (int)blockIdx.x + (g.nfields == 2 ? (k >> 1) : k) * (int)gridDim.x;
#else
    const int fl = k >= nper ? 1 : 0;
    int r = (int)blockIdx.x + (k - fl * nper) * (int)gridDim.x;
#endif
    f = g.f0 + fl;
    c0 = NC == 1 ? r / per_comp : 0;  // single-component tiles: component slowest
    r -= c0 * per_comp;
    o = r / nstrips;
    x0 = (r - o * nstrips) * W;
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < K::NSLOT; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int j = 0; j < K::NSLOT - 1 && j < nmine; ++j) {
      int f, o, x0, c0;
      coords(j, f, o, x0, c0);
      col3_issue(f == 0 ? &tmA : &tmB, smem + j * K::SLOT, &bars[j], x0, col3_outer(g, o), K::TX, c0);
    }
  double2* tws = smem + K::NSLOT * K::SLOT;
  for (int i = threadIdx.x; i < L / 2; i += blockDim.x) tws[tw_swz(i)] = __ldg(&a.tw[g.axis][i]);
  __syncthreads();
  const SmemTw tw{tws};
  const LineSync<T> lsync{1 + line};
  double acc = 0.0;
  for (int k = 0; k < nmine; ++k) {
    const int s = k % K::NSLOT;
    int f, o, x0, c0;
    coords(k, f, o, x0, c0);
    const int comp = NC == 1 ? c0 : lcomp;
    double2* slot = smem + s * K::SLOT;
    mbar_wait(&bars[s], (unsigned)((k / K::NSLOT) & 1));
    double2 v[1][E];
#pragma unroll
    for (int i = 0; i < E; ++i) v[0][i] = slot[K::land(lcomp, pos_first<L, E>(INV_ONLY, t, i), w)];
    // (peer bulk copies: each thread's copies out of the slot reloaded below
    // have been read before thread 0 reloads it)
    if constexpr (PEER) bulk_wait_read0();
    __syncthreads();  // every input is in registers: the slot becomes the lines' exchange scratch
    if (threadIdx.x == 0 && k + K::NSLOT - 1 < nmine) {
      // tile k+NSLOT-1 into the slot of tile k-1, whose store was committed one tile ago
      const int nk = k + K::NSLOT - 1;
      int nf, no, nx0, nc0;
      coords(nk, nf, no, nx0, nc0);
#if FFTC_COL3_PF
      if (nk + 1 < nmine) {  // the tile after it: DRAM -> L2 while this one is transformed
        int pf, po_, px0, pc0;
        coords(nk + 1, pf, po_, px0, pc0);
        col3_prefetch(pf == 0 ? &tmA : &tmB, px0, col3_outer(g, po_));
      }
#endif
      col3_issue(nf == 0 ? &tmA : &tmB, smem + (nk % K::NSLOT) * K::SLOT, &bars[nk % K::NSLOT], nx0, col3_outer(g, no),
                 K::TX, nc0);
    }
    double2* xb = slot + line * K::XS;  // this line's own buffer
    const bool parseval_only = (MODE == MID_EM) && f == 1;
    // (tail barrier -- of the line's threads -- where the projection writes
    // the buffer next; the other paths pass a CTA barrier first)
    if constexpr (!INV_ONLY) fft_line<L, E, 1, false, MID>(v, t, tw, SmemBuf{xb, 0}, lsync);
    if constexpr (MID) {
      // Gamma projection (spectral_ops.py:124-127), k = (kx, k_outer, k_line)
      // for the components (x, y, z).  Each line leaves k_c F^_c in its own
      // buffer (position pos at entry pos); the other two components of the
      // same column read it from there.
      const double kx = (double)wavenum(x0 + w, a.nx), ko = (double)wavenum(g.o0 + o, g.on);
      const double2* b0 = slot + (0 * W + w) * K::XS;
      const double2* b1 = slot + (1 * W + w) * K::XS;
      const double2* b2 = slot + (2 * W + w) * K::XS;
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int pos = pos_last<L, E>(false, t, i);
        const double kc = comp == 0 ? kx : (comp == 1 ? ko : (double)wavenum(pos, L));
        xb[pos] = cscale(v[0][i], kc);
      }
      __syncthreads();
      if (parseval_only) {
        // flux field: only sum_k |Gamma^ j^|^2 / N^2 = sum_k |k.j^|^2 / (|k|^2 N^2)
        // (Parseval, solvers.py:427-430) -- one evaluation per mode, the
        // modes of a thread's E elements dealt round robin over the three
        // component threads that hold them: sum_c |k_c d ik2 / N|^2
        // = |d ik2 / N|^2 |k|^2 with d = k.F^ and ik2 = scale / |k|^2.
        // (No closing barrier: this slot is next written by the TMA load
        // issued after the following tile's input barrier.)
#pragma unroll
        for (int i = 0; i < E; ++i) {
          if (i % 3 != comp) continue;
          const int pos = pos_last<L, E>(false, t, i);
          const double kl = (double)wavenum(pos, L);
          const double k2 = kx * kx + ko * ko + kl * kl;
          const double ik2 = (k2 != 0.0) ? inv_k2(k2) * a.gscale : 0.0;
          const double2 d = cadd(cadd(b0[pos], b1[pos]), b2[pos]);
          acc += cabs2(cscale(d, ik2 * a.inv_n)) * k2;
        }
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int pos = pos_last<L, E>(false, t, i);
          const double kl = (double)wavenum(pos, L);
          const double kc = comp == 0 ? kx : (comp == 1 ? ko : kl);
          const double k2 = kx * kx + ko * ko + kl * kl;
          const double ik2 = (k2 != 0.0) ? inv_k2(k2) * a.gscale : 0.0;
          // k.F^ = (kx Fx + ky Fy) + kz Fz summed in the same order by every
          // component thread; a thread's own term comes from its registers
          // (comp is warp uniform), formed with unfused multiplies so it is
          // the value the other two threads read from the buffer, bit for bit
          const double2 mine = make_double2(__dmul_rn(v[0][i].x, kc), __dmul_rn(v[0][i].y, kc));
          const double2 s0 = comp == 0 ? mine : b0[pos];
          const double2 s1 = comp == 1 ? mine : b1[pos];
          const double2 s2 = comp == 2 ? mine : b2[pos];
          double2 dot = cadd(cadd(s0, s1), s2);
          dot = cscale(dot, ik2);
          if (MODE == MID_BASIC) {
            const double2 gc = cscale(dot, kc);
            acc += cabs2(cscale(gc, a.inv_n));  // Parseval on the 1/N-scaled mode
            v[0][i] = gc;
          } else {
            v[0][i] = csub(v[0][i], cscale(dot, 2.0 * kc));
          }
        }
        __syncthreads();  // k.F^ reads are done before the inverse transform's exchanges
      }
    }
    if (!parseval_only) {
      // (the CTA barrier below orders the inverse's last exchange reads)
      if constexpr (MODE != COL_FWD) fft_line<L, E, 1, true, false>(v, t, tw, SmemBuf{xb, 0}, lsync);
      __syncthreads();  // every line's exchange reads are done before outputs overwrite the slot
      const bool inv_layout = (MODE != COL_FWD);
      if constexpr (PEER) {
        // Outputs staged dense [c][pos][w], then one bulk copy per (component,
        // line position): the tile's W adjacent x-values are one contiguous
        // 16W-byte run in the owning rank's slab (NVLink to peers).
#pragma unroll
        for (int i = 0; i < E; ++i) slot[(lcomp * L + pos_last<L, E>(inv_layout, t, i)) * W + w] = v[0][i];
        fence_proxy_async();
        __syncthreads();
        const int rq = po->rows_per_rank;
        for (int r = threadIdx.x; r < NC * L; r += (int)blockDim.x) {
          const int lc = r / L, pos = r - lc * L;
          const int cc = NC == 1 ? comp : lc;
          const int q = pos / rq;
          const long long p = pos - q * rq;
          long long off;
          if (po->zs > 0) {  // z-blocked destination slabs
            const int zs = po->zs;
            const long long O = po->outer0 + o;
            const long long b = po->blk_line ? p : O, u = po->blk_line ? O : p;
            const long long row = (((b >> zs) * po->bn + u) << zs) | (b & ((1 << zs) - 1));
            off = cc * po->comp_stride + x0 + row * po->row_len;
          } else {
            off = cc * po->comp_stride + (po->outer0 + o) * po->outer_stride + x0 + p * po->line_stride;
          }
          bulk_s2g(po->dst[f][q] + off, slot + (lc * L + pos) * W, (unsigned)(W * sizeof(double2)));
        }
        bulk_commit();
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i) slot[K::land(lcomp, pos_last<L, E>(inv_layout, t, i), w)] = v[0][i];
        fence_proxy_async();
        __syncthreads();
        if (threadIdx.x == 0) {
          col3_store(f == 0 ? &tmA : &tmB, slot, x0, col3_outer(g, o), c0);
          bulk_commit();
        }
      }
    }
  }
  if (threadIdx.x == 0 || PEER) bulk_wait0();  // stores have landed in global memory
  if constexpr (PEER) __threadfence_system();  // peer stores visible before the host-level barrier
  if constexpr (MID) {
    double in[1] = {acc}, tot[1];
    if (grid_reduce<1>(in, tot, a) && threadIdx.x == 0 && !a.op_mode && !g.no_monitor) {
      if (a.dist) a.st->parseval = tot[0] / a.inv_n;
      else monitor_step(a, tot[0] / a.inv_n + a.st->js2);
    }
  }
}

// ----------------------------------------------------------------------------
// The z pass with the projection, three components per thread.
//
// In k_col3_lg a thread owns one component of one column, so the projection's
// k.F^ has to cross threads through shared memory: 3 of the A tile's 15
// shared-memory passes (ncu: the pass runs at ~75 % of the shared-memory
// wavefront rate, FP64 ~45 %).  Here a thread carries all three components of
// its 8 line positions through the transforms (fft_line with C = 3 channels:
// one set of twiddle powers serves the three), the projection is thread
// local -- no exchange, no CTA barrier -- and a tile costs 12 passes instead
// of 15 (flux tiles 6 instead of 8).  256 threads per CTA (W columns x T),
// a column's T threads synchronise among themselves in the transforms.
// ----------------------------------------------------------------------------
template <int L>
struct Col3Mid {
  using G = Col3Lg<L>;
  static constexpr int E = G::E, T = G::T, W = G::W, NC = 3;
  static constexpr int THREADS = W * T;
  static constexpr int XS = G::XS, SLOT = G::SLOT, NSLOT = G::NSLOT, SMEM = G::SMEM;
  static constexpr unsigned TX = G::TX;
};

template <int MODE, int L, bool PEER = false>
__global__ void __launch_bounds__(Col3Mid<L>::THREADS, 1)
    k_col3_mid(Args a, Line3 g, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const PeerOut* __restrict__ po) {
  using K = Col3Mid<L>;
  using KG = Col3Lg<L>;
  constexpr int E = K::E, T = K::T, W = K::W, NC = K::NC;
  constexpr bool MID = (MODE == MID_BASIC || MODE == MID_EM);  // else a plain y pass, three components per thread
  constexpr bool INV_ONLY = (MODE == COL_INV);
  extern __shared__ __align__(128) double2 smem_raw[];
  __shared__ uint64_t bars[K::NSLOT];
  if (!a.op_mode && a.st->stopped) return;
  double2* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u) / (unsigned)sizeof(double2);
  const int t = threadIdx.x % T, w = threadIdx.x / T;
  const int nstrips = a.nx / W;
  const int per_field = g.nouter * nstrips;
  const int nper = (int)blockIdx.x < per_field ? (per_field - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  const int nmine = nper * g.nfields;
  auto coords = [&](int k, int& f, int& o, int& x0) {  // (as k_col3_lg: per-field round robin, A/B alternating)
#if FFTC_COL3_ALT
    const int fl = g.nfields == 2 ? (k & 1) : 0;
    const int r = (int)blockIdx.x + (g.nfields == 2 ? (k >> 1) : k) * (int)gridDim.x;
#else
    const int fl = k >= nper ? 1 : 0;
    const int r = (int)blockIdx.x + (k - fl * nper) * (int)gridDim.x;
#endif
    f = g.f0 + fl;
    o = r / nstrips;
    x0 = (r - o * nstrips) * W;
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < K::NSLOT; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int j = 0; j < K::NSLOT - 1 && j < nmine; ++j) {
      int f, o, x0;
      coords(j, f, o, x0);
      col3_issue(f == 0 ? &tmA : &tmB, smem + j * K::SLOT, &bars[j], x0, col3_outer(g, o), K::TX);
    }
  double2* tws = smem + K::NSLOT * K::SLOT;
  for (int i = threadIdx.x; i < L / 2; i += blockDim.x) tws[tw_swz(i)] = __ldg(&a.tw[g.axis][i]);
  __syncthreads();
  const SmemTw tw{tws};
  const LineSync<T> lsync{1 + w};
  double acc = 0.0;
  for (int k = 0; k < nmine; ++k) {
    const int s = k % K::NSLOT;
    int f, o, x0;
    coords(k, f, o, x0);
    double2* slot = smem + s * K::SLOT;
    mbar_wait(&bars[s], (unsigned)((k / K::NSLOT) & 1));
    double2 v[NC][E];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int i = 0; i < E; ++i) v[c][i] = slot[KG::land(c, pos_first<L, E>(INV_ONLY, t, i), w)];
    if constexpr (PEER) bulk_wait_read0();
    __syncthreads();  // every input is in registers: the slot becomes the columns' exchange scratch
    if (threadIdx.x == 0 && k + K::NSLOT - 1 < nmine) {
      const int nk = k + K::NSLOT - 1;
      int nf, no, nx0;
      coords(nk, nf, no, nx0);
      col3_issue(nf == 0 ? &tmA : &tmB, smem + (nk % K::NSLOT) * K::SLOT, &bars[nk % K::NSLOT], nx0, col3_outer(g, no),
                 K::TX);
    }
    // channel c of column w transforms in the buffer (c, w) of the slot
    const SmemBuf xb{slot + w * K::XS, W * K::XS};
    const bool parseval_only = (MODE == MID_EM) && f == 1;
    // (no tail barrier: the projection touches no shared memory, and the
    // inverse's first exchange is preceded by the column barrier below)
    if constexpr (!INV_ONLY) fft_line<L, E, NC, false, false>(v, t, tw, xb, lsync);
    if constexpr (MID) {
    // Gamma projection (spectral_ops.py:124-127), k = (kx, k_outer, k_line)
    const double kx = (double)wavenum(x0 + w, a.nx), ko = (double)wavenum(g.o0 + o, g.on);
    const double kxo2 = kx * kx + ko * ko;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int pos = pos_last<L, E>(false, t, i);
      const double kl = (double)wavenum(pos, L);
      const double k2 = fma(kl, kl, kxo2);
      const double ik2 = (k2 != 0.0) ? inv_k2(k2) * a.gscale : 0.0;
      // k.F^ = (kx Fx + ky Fy) + kz Fz, unfused products like the exchanged form
      double2 dot;
      dot.x = (__dmul_rn(v[0][i].x, kx) + __dmul_rn(v[1][i].x, ko)) + __dmul_rn(v[2][i].x, kl);
      dot.y = (__dmul_rn(v[0][i].y, kx) + __dmul_rn(v[1][i].y, ko)) + __dmul_rn(v[2][i].y, kl);
      if (parseval_only) {
        // flux field: sum_k |Gamma^ j^|^2 / N^2 = sum_k |k.j^|^2 / (|k|^2 N^2)
        // (Parseval, solvers.py:427-430), one evaluation per mode
        acc += cabs2(cscale(dot, ik2 * a.inv_n)) * k2;
      } else {
        dot = cscale(dot, ik2);
        if (MODE == MID_BASIC) {
          const double2 g0 = cscale(dot, kx), g1 = cscale(dot, ko), g2 = cscale(dot, kl);
          acc += cabs2(cscale(g0, a.inv_n)) + cabs2(cscale(g1, a.inv_n)) + cabs2(cscale(g2, a.inv_n));
          v[0][i] = g0;
          v[1][i] = g1;
          v[2][i] = g2;
        } else {  // (I - 2 Gamma^) F
          v[0][i] = csub(v[0][i], cscale(dot, 2.0 * kx));
          v[1][i] = csub(v[1][i], cscale(dot, 2.0 * ko));
          v[2][i] = csub(v[2][i], cscale(dot, 2.0 * kl));
        }
      }
    }
    }  // MID
    if (!parseval_only) {
      if constexpr (MID) lsync();  // the column's last forward exchange reads are done
      if constexpr (MODE != COL_FWD) fft_line<L, E, NC, true, false>(v, t, tw, xb, lsync);
      constexpr bool inv_layout = (MODE != COL_FWD);
      __syncthreads();  // every column's exchange reads are done before outputs overwrite the slot
      if constexpr (PEER) {
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int i = 0; i < E; ++i) slot[(c * L + pos_last<L, E>(inv_layout, t, i)) * W + w] = v[c][i];
        fence_proxy_async();
        __syncthreads();
        const int rq = po->rows_per_rank;
        for (int r = threadIdx.x; r < 3 * L; r += (int)blockDim.x) {
          const int cc = r / L, pos = r - cc * L;
          const int q = pos / rq;
          const long long p = pos - q * rq;
          long long off;
          if (po->zs > 0) {  // z-blocked destination slabs
            const int zs = po->zs;
            const long long O = po->outer0 + o;
            const long long b = po->blk_line ? p : O, u = po->blk_line ? O : p;
            const long long row = (((b >> zs) * po->bn + u) << zs) | (b & ((1 << zs) - 1));
            off = cc * po->comp_stride + x0 + row * po->row_len;
          } else {
            off = cc * po->comp_stride + (po->outer0 + o) * po->outer_stride + x0 + p * po->line_stride;
          }
          bulk_s2g(po->dst[f][q] + off, slot + (cc * L + pos) * W, (unsigned)(W * sizeof(double2)));
        }
        bulk_commit();
      } else {
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int i = 0; i < E; ++i) slot[KG::land(c, pos_last<L, E>(inv_layout, t, i), w)] = v[c][i];
        fence_proxy_async();
        __syncthreads();
        if (threadIdx.x == 0) {
          col3_store(f == 0 ? &tmA : &tmB, slot, x0, col3_outer(g, o));
          bulk_commit();
        }
      }
    }
    // (flux tiles: this slot is next written by the TMA load issued after the
    // following tile's input barrier, which every thread reaches after its
    // last exchange read here)
  }
  if (threadIdx.x == 0 || PEER) bulk_wait0();  // stores have landed in global memory
  if constexpr (PEER) __threadfence_system();  // peer stores visible before the host-level barrier
  if constexpr (MID) {
    double in[1] = {acc}, tot[1];
    if (grid_reduce<1>(in, tot, a) && threadIdx.x == 0 && !a.op_mode && !g.no_monitor) {
      if (a.dist) a.st->parseval = tot[0] / a.inv_n;
      else monitor_step(a, tot[0] / a.inv_n + a.st->js2);
    }
  }
}

}  // namespace fftc
