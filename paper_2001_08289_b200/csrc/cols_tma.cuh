// cols_tma.cuh -- TMA tensor-map staged 2-D projection sweep (sweep 2).
//
// Line = one x-column of one work field (A: the EM residual field R / the
// flux of basic-type schemes; B: the flux J, Parseval only), both vector
// components.  The column is strided in HBM (pitch nx*16 B), so it is fetched
// with cp.async.bulk.tensor (a 3-D tensor map {2*nx doubles, ny, d}, boxes of
// 256 rows x 16 B) into a ring of 3 shared-memory slots completed on
// mbarriers.  The CTA has two halves of 2*T threads; each half processes
// every other line, so two lines are in compute while the third streams in.
// A slot doubles as the line's FFT exchange buffer once its data is in
// registers.  Per element: y-FFT (radix 16, two exchanges), the Gamma_1
// projection with the partner component in lane^16 (spectral_ops.py:124-127),
// Parseval residual accumulation, y-iFFT and a direct store.
#pragma once
#include <cuda.h>

#include "sweeps.cuh"

namespace fftc {

template <int L>
struct ColTma {
  static constexpr int E = 16;
  static constexpr int T = L / E;
  static constexpr int HALF = 2 * T;  // (component, t) pairs of one line
  static constexpr int THREADS = 2 * HALF;
  static constexpr int LP = Plan<L, E>::LP;
  static constexpr int NSLOT = 3;
  static constexpr int CB = LP + 8;         // exchange buffer stride per component
  static constexpr int SLOT = 2 * CB + 8;   // double2 units: two skewed exchange buffers (>= 2L TMA landing)
  // + twiddle copy: load_twbase only reads indices (R/2)*m < L/2 (m < L/R)
  static constexpr int SMEM = (NSLOT * SLOT + L / 2) * (int)sizeof(double2);
  static_assert(SMEM <= 232448 - 64, "column kernel exceeds the 227 KB dynamic shared memory limit");
  static constexpr int BOXR = L < 256 ? L : 256;  // rows per TMA box
  static constexpr unsigned TX = (unsigned)(2 * L * sizeof(double2));
  // one CTA per SM at L = 2048 (the ring fills shared memory); shorter
  // columns fit several CTAs, up to 16 warps per SM
  static constexpr int MINB_FILL = (232448 / (SMEM + 2048)) < (512 / THREADS) ? (232448 / (SMEM + 2048)) : (512 / THREADS);
  static constexpr int MINB = MINB_FILL > 1 ? MINB_FILL : 1;
};

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* tm, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(tm),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// One tensor copy brings both components of column x, all L rows: the map is
// 4-D {2 doubles, BOXR rows, L/BOXR row blocks, d components}, box
// {2, BOXR, L/BOXR, 2}, landing dense as [comp][y] in the slot.
template <int L>
__device__ __forceinline__ void cols_tma_issue(const CUtensorMap* tm, double2* slot, uint64_t* bar, int x) {
  using K = ColTma<L>;
  bulk_wait_read0();  // an earlier TMA store from this slot has finished reading it
  mbar_expect_tx(bar, K::TX);
  tma_load_4d(slot, tm, 2 * x, 0, 0, 0, bar);
}

#ifdef FFTC_PHASE_TIMING
#define PHASE_MARK(i)                                                                            \
  do {                                                                                           \
    const long long now_ = clock64();                                                            \
    if (ht == 0 && a.dbg) atomicAdd(&a.dbg[i], (unsigned long long)(now_ - tph_));               \
    tph_ = now_;                                                                                 \
  } while (0)
#else
#define PHASE_MARK(i) \
  do {                \
  } while (0)
#endif

template <int MODE, int L>
__global__ void __launch_bounds__(ColTma<L>::THREADS, ColTma<L>::MINB)
    k_mid2_tma(Args a, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB) {
  using K = ColTma<L>;
  constexpr int E = K::E;
  constexpr int NQ = 1;
  extern __shared__ __align__(128) double2 smem[];
  // bars: slot s holds line k's data (TMA complete_tx).  cbars: the half that
  // consumed line k has released slot s.  The two halves take lines k = half,
  // half+2, ... and share the NSLOT-ring, so line k reuses the slot of line
  // k-NSLOT, consumed by the other half.  A half may run ahead (the EM scheme's
  // parseval-only lines skip the inverse FFT and the store); without cbars its
  // parity wait for line k could alias line k-2*NSLOT's completed phase while
  // line k-NSLOT's copy is still in flight.
  __shared__ uint64_t bars[K::NSLOT], cbars[K::NSLOT];
  if (!a.op_mode && a.st->stopped) return;
  const int half = threadIdx.x / K::HALF, ht = threadIdx.x % K::HALF;
  // component in lane bit CB (16 lanes of one component side by side): an
  // 8-lane LDS.128 phase then reads 128 contiguous bytes of one component
  // instead of two components whose [comp][y] landing rows share banks
  constexpr int CB = K::T >= 16 ? 4 : (K::T >= 8 ? 3 : (K::T >= 4 ? 2 : (K::T >= 2 ? 1 : 0)));
  const int comp = (ht >> CB) & 1, t = (ht & ((1 << CB) - 1)) | ((ht >> (CB + 1)) << CB);
  const HalfSync hsync{1 + half, K::HALF};
  const int nfields = (MODE == MID_EM) ? 2 : 1;
  // 32-bit line bookkeeping (nx <= 4096): the loop state stays in registers
  const int lines = a.nx * nfields;
  const int nmine = (int)blockIdx.x < lines ? (lines - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < K::NSLOT; ++s) {
      mbar_init(&bars[s], 1);
      mbar_init(&cbars[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = 0; s < K::NSLOT && s < nmine; ++s) {
      const int line = (int)blockIdx.x + s * (int)gridDim.x;
      const int f = line / a.nx;
      cols_tma_issue<L>(f == 0 ? &tmA : &tmB, smem + s * K::SLOT, &bars[s], line - f * a.nx);
    }
  double2* tws = smem + K::NSLOT * K::SLOT;
  for (int i = threadIdx.x; i < L / 2; i += blockDim.x) tws[tw_swz(i)] = __ldg(&a.tw[1][i]);
  __syncthreads();
  const SmemTw twy{tws};
  const double tdbl = (double)t;  // (ny == L: this kernel's columns span the grid)
  const double g2 = 2.0 * a.gscale;
  double acc[NQ] = {0.0};
#ifdef FFTC_PHASE_TIMING
  long long tph_ = clock64();
#endif
  for (int k = half; k < nmine; k += 2) {
    const int s = k % K::NSLOT;
    const int line = (int)blockIdx.x + k * (int)gridDim.x;
    const int f = line / a.nx;
    const int x = line - f * a.nx;
    double2* slot = smem + s * K::SLOT;
    const double2* inb = slot + comp * L;  // TMA landing layout [comp][y]
    // exchange buffers: component c at c*CB, component 1 skewed by 4 slots
    // (64 B) so that partner lanes hit disjoint bank groups
    double2* xbuf = slot + comp * (K::CB + 4);
    PHASE_MARK(0);
    static_assert(K::NSLOT % 2 == 1, "line k-NSLOT must belong to the other half");
    if (k >= K::NSLOT) mbar_wait(&cbars[s], (unsigned)((k / K::NSLOT - 1) & 1));
    mbar_wait(&bars[s], (unsigned)((k / K::NSLOT) & 1));
    PHASE_MARK(1);
    double2 v[1][E];
#pragma unroll
    for (int i = 0; i < E; ++i) v[0][i] = inb[pos_first<L, E>(false, t, i)];
    hsync();  // slot becomes exchange scratch
    PHASE_MARK(2);
    fft_line<L, E, 1, false>(v, t, twy, SmemBuf{xbuf, 0}, hsync);
    PHASE_MARK(3);
    const double kx = (double)wavenum(x, a.nx);
    const double kx2 = kx * kx;
    const bool parseval_only = (MODE == MID_EM) && f == 1;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      // element i sits at y = t + off_i (off_i a multiple of T, fixed at
      // compile time), so its wave number is t + (off_i or off_i - L): one
      // add to the thread's converted index instead of a conversion per element
      const int off = pos_last<L, E>(false, 0, i);
      const double ky = tdbl + (double)(off >= L / 2 ? off - L : off);
      const double kc = comp ? ky : kx;
      const double k2 = fma(ky, ky, kx2);
      const double ik2 = (k2 != 0.0) ? inv_k2(k2) : 0.0;
      const double2 mine = cscale(v[0][i], kc);
      double2 other;
      other.x = __shfl_xor_sync(0xffffffffu, mine.x, 1 << CB);
      other.y = __shfl_xor_sync(0xffffffffu, mine.y, 1 << CB);
      const double2 dot = comp ? cadd(other, mine) : cadd(mine, other);  // kx F_x + ky F_y
      // one real weight per element: (Gamma^ F)_c = w dot, w = k_c |k|^-2 scale
      if (MODE == MID_BASIC || parseval_only) {
        const double2 g = cscale(dot, kc * ik2 * a.gscale);
        acc[0] += cabs2(cscale(g, a.inv_n));
        v[0][i] = g;
      } else {  // (I - 2 Gamma^) F
        const double w = kc * ik2 * g2;
        v[0][i] = make_double2(fma(-w, dot.x, v[0][i].x), fma(-w, dot.y, v[0][i].y));
      }
    }
    PHASE_MARK(4);
    if (!parseval_only) {
      // (no tail barrier: the hsync below orders the last exchange reads)
      fft_line<L, E, 1, true, false>(v, t, twy, SmemBuf{xbuf, 0}, hsync);
      PHASE_MARK(5);
      // outputs -> slot in the tensor layout, then one TMA store per line;
      // the barrier first: another warp of this half may still be reading its
      // last exchange from padded addresses the dense outputs overwrite
      hsync();
      double2* outb = slot + comp * L;
#pragma unroll
      for (int i = 0; i < E; ++i) outb[pos_last<L, E>(true, t, i)] = v[0][i];
      fence_proxy_async();
      hsync();
      if (ht == 0) {
        tma_store_4d(&tmA, slot, 2 * x, 0, 0, 0);
        bulk_commit();
      }
    }  // parseval-only lines: the forward transform's tail barrier was the slot's last use
    PHASE_MARK(6);
    if (ht == 0) mbar_arrive(&cbars[s]);  // after the hsync above: every thread of this half is done with slot s
    if (ht == 0 && k + K::NSLOT < nmine) {
      fence_proxy_async();
      const int nl = line + K::NSLOT * (int)gridDim.x;
      const int nf = nl / a.nx;
      cols_tma_issue<L>(nf == 0 ? &tmA : &tmB, smem + s * K::SLOT, &bars[s], nl - nf * a.nx);
      PHASE_MARK(7);
    }
  }
  if (ht == 0) bulk_wait0();  // this half's TMA stores have landed in global memory
  double tot[NQ];
  if (grid_reduce<NQ>(acc, tot, a) && threadIdx.x == 0 && !a.op_mode) {
    if (a.dist) a.st->parseval = tot[0] / a.inv_n;
    else monitor_step(a, tot[0] / a.inv_n + a.st->js2);
  }
}

}  // namespace fftc
