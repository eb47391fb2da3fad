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
// projection with the partner component in lane^1 (spectral_ops.py:124-127),
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
  static constexpr int CB = LP + 8;    // component buffer (128-B aligned for TMA)
  static constexpr int SLOT = 2 * CB;  // double2 units, two components
  static constexpr int SMEM = NSLOT * SLOT * (int)sizeof(double2);
  static constexpr int BOXR = L < 256 ? L : 256;  // rows per TMA box
  static constexpr unsigned TX = (unsigned)(2 * L * sizeof(double2));
};

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

template <int L>
__device__ __forceinline__ void cols_tma_issue(const CUtensorMap* tm, double2* slot, uint64_t* bar, int x) {
  using K = ColTma<L>;
  mbar_expect_tx(bar, K::TX);
#pragma unroll 1
  for (int c = 0; c < 2; ++c)
#pragma unroll 1
    for (int y0 = 0; y0 < L; y0 += K::BOXR) tma_load_3d(slot + c * K::CB + y0, tm, 2 * x, y0, c, bar);
}

struct HalfSync {
  int id;
  int n;
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
};

template <int MODE, int L>
__global__ void __launch_bounds__(ColTma<L>::THREADS, 1)
    k_mid2_tma(Args a, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB) {
  using K = ColTma<L>;
  constexpr int E = K::E;
  constexpr int NQ = 1;
  extern __shared__ __align__(128) double2 smem[];
  __shared__ uint64_t bars[K::NSLOT];
  if (!a.op_mode && a.st->stopped) return;
  const int half = threadIdx.x / K::HALF, ht = threadIdx.x % K::HALF;
  const int comp = ht & 1, t = ht >> 1;
  const HalfSync hsync{1 + half, K::HALF};
  const int nfields = (MODE == MID_EM) ? 2 : 1;
  const long long lines = (long long)a.nx * nfields;
  const long long nmine = blockIdx.x < lines ? (lines - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < K::NSLOT; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = 0; s < K::NSLOT && s < nmine; ++s) {
      const long long line = blockIdx.x + (long long)s * gridDim.x;
      const int f = (int)(line / a.nx);
      cols_tma_issue<L>(f == 0 ? &tmA : &tmB, smem + s * K::SLOT, &bars[s], (int)(line - (long long)f * a.nx));
    }
  double acc[NQ] = {0.0};
  for (long long k = half; k < nmine; k += 2) {
    const int s = (int)(k % K::NSLOT);
    const long long line = blockIdx.x + k * gridDim.x;
    const int f = (int)(line / a.nx);
    const int x = (int)(line - (long long)f * a.nx);
    double2* buf = smem + s * K::SLOT + comp * K::CB;
    // exchanges of component 1 run 4 slots (64 B) off component 0: the
    // partner lanes then hit disjoint bank groups
    double2* xbuf = buf + 4 * comp;
    mbar_wait(&bars[s], (unsigned)((k / K::NSLOT) & 1));
    double2 v[1][E];
#pragma unroll
    for (int i = 0; i < E; ++i) v[0][i] = buf[pos_first<L, E>(false, t, i)];
    hsync();  // slot becomes exchange scratch
    fft_line<L, E, 1, false>(v, t, a.tw[1], SmemBuf{xbuf, 0}, hsync);
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
      other.x = __shfl_xor_sync(0xffffffffu, mine.x, 1);
      other.y = __shfl_xor_sync(0xffffffffu, mine.y, 1);
      double2 dot = comp ? cadd(other, mine) : cadd(mine, other);  // kx F_x + ky F_y
      dot = cscale(dot, ik2);
      if (MODE == MID_BASIC || parseval_only) {
        const double2 g = cscale(dot, kc);
        acc[0] += cabs2(cscale(g, a.inv_n));
        v[0][i] = g;
      } else {
        v[0][i] = csub(v[0][i], cscale(dot, 2.0 * kc));
      }
    }
    if (!parseval_only) {
      fft_line<L, E, 1, true>(v, t, a.tw[1], SmemBuf{xbuf, 0}, hsync);
      double2* F = ((f == 0) ? a.A : a.B) + (size_t)comp * a.N + x;
#pragma unroll
      for (int i = 0; i < E; ++i) F[(size_t)pos_last<L, E>(true, t, i) * a.nx] = v[0][i];
    }
    hsync();  // slot s consumed
    if (ht == 0 && k + K::NSLOT < nmine) {
      fence_proxy_async();
      const long long nl = line + (long long)K::NSLOT * gridDim.x;
      const int nf = (int)(nl / a.nx);
      cols_tma_issue<L>(nf == 0 ? &tmA : &tmB, smem + s * K::SLOT, &bars[s], (int)(nl - (long long)nf * a.nx));
    }
  }
  double tot[NQ];
  if (grid_reduce<NQ>(acc, tot, a) && threadIdx.x == 0 && !a.op_mode)
    monitor_step(a, tot[0] * (double)a.N + a.st->js2);
}

}  // namespace fftc
