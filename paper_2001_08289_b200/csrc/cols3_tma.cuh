// cols3_tma.cuh -- TMA-staged column passes of 3-D fields (the y passes and
// the z pass with the Gamma projection) for line lengths 256..1024.
//
// Same algebra as k_col (sweeps.cuh): the 3-D Gamma_1 of
// spectral_ops.py:120-128 (a third wave-vector component) and the plain y
// transforms around it.  Data movement:
//   * a tile is W adjacent x-columns of all three components along the
//     line axis; ONE cp.async.bulk.tensor copy of a 5-D tensor map {2*nx
//     doubles, 256-row block, L/256 blocks, outer index, component} with box
//     {2W, 256, L/256, 1, 3} lands it in shared memory as [c][pos][w] --
//     whatever the line stride (z: nx*ny, y: nx).  W is chosen so a box row
//     is 64..128 B: one-column boxes (16 B rows) run into the TMA request
//     rate and, along z, touch a new 2 MB page per 16 bytes;
//   * one tile per CTA at a time (3*W*T = 768 threads, radix 8, 16 data
//     registers per thread), two slots: tile j+1 streams in while tile j is
//     transformed, tile j leaves by TMA store while tile j+1 starts;
//   * the slot is the FFT exchange area once the inputs are in registers;
//     the projection's k.F^ crosses the component warps through it.
// Tiles are numbered x fastest, so concurrent CTAs work on neighbouring
// columns of the same rows.
#pragma once
#include "cols_tma.cuh"
#include "kernel_table.h"

namespace fftc {

template <int L>
struct Col3Tma {
  static constexpr int E = 8;
  static constexpr int T = L / E;
  static constexpr int W = col3_tile_w(L);  // columns per tile
  static constexpr int NC = 3;
  static constexpr int THREADS = NC * W * T;
  static constexpr int LP = Plan<L, E>::LP;
  // per (component, column) exchange stride: the W buffers start in distinct
  // 16-B bank groups, and SLOT stays a multiple of 8 entries (128 B)
  static constexpr int XS = LP + (W == 2 ? 4 : 2);
  static constexpr int SLOT = NC * W * XS;  // >= NC*W*L landing
#ifndef FFTC_COL3_NSLOT
#define FFTC_COL3_NSLOT 2
#endif
  static constexpr int NSLOT_FIT = (232448 - 512 - (L / 2) * 16) / (SLOT * 16);
  // tiles in flight + the one being transformed (as many as fit, up to FFTC_COL3_NSLOT)
  static constexpr int NSLOT = FFTC_COL3_NSLOT < NSLOT_FIT ? FFTC_COL3_NSLOT : NSLOT_FIT;
  static constexpr int SMEM = (NSLOT * SLOT + L / 2) * (int)sizeof(double2);
  static constexpr int BOXR = L < 256 ? L : 256;
  static constexpr unsigned TX = (unsigned)(NC * W * L * sizeof(double2));
  // narrow tiles (384 threads) leave room for two CTAs per SM: registers for both
  static constexpr int MINB = THREADS <= 384 ? 2 : 1;
  static_assert(THREADS <= 1024, "block size");
  static_assert((SLOT * 16) % 128 == 0, "TMA destinations stay 128-B aligned");
  static_assert(SMEM <= 232448 - 512, "shared memory budget");
};

// tensor-map coordinates (dims 2 and 3) of outer line o (Line3::obs/om)
__device__ __forceinline__ int2 col3_outer(const Line3& g, int o) {
  return g.om > 0 ? make_int2((o >> g.obs) * g.om, o & ((1 << g.obs) - 1)) : make_int2(0, o);
}
__device__ __forceinline__ void col3_issue(const CUtensorMap* tm, double2* slot, uint64_t* bar, int x0, int2 oc,
                                           unsigned tx, int c0 = 0) {
  bulk_wait_read0();  // the TMA store that last used this slot has read it out
  mbar_expect_tx(bar, tx);
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
      "%6}], [%7];" ::"r"(smem_u32(slot)),
      "l"(tm), "r"(2 * x0), "r"(0), "r"(oc.x), "r"(oc.y), "r"(c0), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void col3_store(const CUtensorMap* tm, const double2* slot, int x0, int2 oc, int c0 = 0) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(tm),
               "r"(2 * x0), "r"(0), "r"(oc.x), "r"(oc.y), "r"(c0), "r"(smem_u32(slot))
               : "memory");
}

#ifndef FFTC_PEER_BULK
#define FFTC_PEER_BULK 1
#endif
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}

// PEER: outputs are written straight to their owning rank (PeerOut po,
// device memory) instead of back through the slot and a TMA store -- the
// decomposed solve's transposes fused into the pass that produces the data.
template <int MODE, int L, bool PEER = false>
__global__ void __launch_bounds__(Col3Tma<L>::THREADS, Col3Tma<L>::MINB)
    k_col3_tma(Args a, Line3 g, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const PeerOut* __restrict__ po) {
  using K = Col3Tma<L>;
  constexpr int E = K::E, T = K::T, W = K::W;
  constexpr bool MID = (MODE == MID_BASIC || MODE == MID_EM);
  constexpr bool INV_ONLY = (MODE == COL_INV);
  extern __shared__ __align__(128) double2 smem[];
  __shared__ uint64_t bars[K::NSLOT];
  if (!a.op_mode && a.st->stopped) return;
  const int w = threadIdx.x % W, t = (threadIdx.x / W) % T, comp = threadIdx.x / (W * T);
  const int nstrips = a.nx / W;
  // 32-bit tile bookkeeping (at most 2 * 4096 * 4096 / W tiles): 64-bit loop
  // state spilled in the 2-D projection sweep, keep it out of the registers here
  const int per_field = g.nouter * nstrips;
  const int tiles = per_field * g.nfields;
  const int nmine = (int)blockIdx.x < tiles ? (tiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  auto coords = [&](int k, int& f, int& o, int& x0) {
    const int tile = (int)blockIdx.x + k * (int)gridDim.x;
    const int fl = tile / per_field;
    const int r = tile - fl * per_field;
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
  double acc = 0.0;
  for (int k = 0; k < nmine; ++k) {
    const int s = k % K::NSLOT;
    int f, o, x0;
    coords(k, f, o, x0);
    double2* slot = smem + s * K::SLOT;
    mbar_wait(&bars[s], (unsigned)((k / K::NSLOT) & 1));
    double2 v[1][E];
#pragma unroll
    for (int i = 0; i < E; ++i) v[0][i] = slot[(comp * L + pos_first<L, E>(INV_ONLY, t, i)) * W + w];
    // (peer bulk copies: each thread's copies out of the other slot have been
    // read before thread 0 reloads it below)
    if constexpr (PEER && FFTC_PEER_BULK) bulk_wait_read0();
    __syncthreads();  // every input is in registers: the slot becomes exchange scratch
    if (threadIdx.x == 0 && k + K::NSLOT - 1 < nmine) {
      // tile k+NSLOT-1 into the slot of tile k-1, whose store was committed one tile ago
      const int nk = k + K::NSLOT - 1;
      const int ns = nk % K::NSLOT;
      int nf, no, nx0;
      coords(nk, nf, no, nx0);
      col3_issue(nf == 0 ? &tmA : &tmB, smem + ns * K::SLOT, &bars[ns], nx0, col3_outer(g, no), K::TX);
    }
    double2* xb = slot + (comp * W + w) * K::XS;
    const bool parseval_only = (MODE == MID_EM) && f == 1;
    // (tail barrier only where the projection needs it; the other paths pass
    // their own barrier before the slot is written again)
    if constexpr (!INV_ONLY) fft_line<L, E, 1, false, MID>(v, t, tw, SmemBuf{xb, 0}, SyncAll{});
    if constexpr (MID) {
      // Gamma projection (spectral_ops.py:124-127), k = (kx, k_outer, k_line)
      // for the components (x, y, z); k.F^ gathered across the component warps.
      // (The forward transform's tail barrier already ordered its last
      // exchange reads before these writes.)
      const double kx = (double)wavenum(x0 + w, a.nx), ko = (double)wavenum(g.o0 + o, g.on);
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int pos = pos_last<L, E>(false, t, i);
        const double kc = comp == 0 ? kx : (comp == 1 ? ko : (double)wavenum(pos, L));
        slot[(comp * L + pos) * W + w] = cscale(v[0][i], kc);
      }
      __syncthreads();
      if (parseval_only) {
        // flux field: only sum_k |Gamma^ j^|^2 / N^2 = sum_k |k.j^|^2 / (|k|^2 N^2)
        // (Parseval, solvers.py:427-430) -- one evaluation per mode, the
        // modes of a thread's E elements dealt round robin over the three
        // component threads that hold them: sum_c |k_c d ik2 / N|^2
        // = |d ik2 / N|^2 |k|^2 with d = k.F^ and ik2 = scale / |k|^2.
#pragma unroll
        for (int i = 0; i < E; ++i) {
          if (i % 3 != comp) continue;
          const int pos = pos_last<L, E>(false, t, i);
          const double kl = (double)wavenum(pos, L);
          const double k2 = kx * kx + ko * ko + kl * kl;
          const double ik2 = (k2 != 0.0) ? inv_k2(k2) * a.gscale : 0.0;
          const double2 d = cadd(cadd(slot[pos * W + w], slot[(L + pos) * W + w]), slot[(2 * L + pos) * W + w]);
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
          // k.F^ = (kx Fx + ky Fy) + kz Fz in the same order on every component
          // thread; a thread's own term comes from its registers (comp is warp
          // uniform), the other two from the slot
          const double2 mine = cscale(v[0][i], kc);
          const double2 s0 = comp == 0 ? mine : slot[pos * W + w];
          const double2 s1 = comp == 1 ? mine : slot[(L + pos) * W + w];
          const double2 s2 = comp == 2 ? mine : slot[(2 * L + pos) * W + w];
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
      }
      __syncthreads();  // kf reads are done before the inverse transform's exchanges (or the next tile)
    }
    if (PEER && !parseval_only) {
#if FFTC_PEER_BULK
      // Outputs staged dense in the slot ([c][pos][w], as for the TMA store),
      // then one bulk copy per (component, line position): the tile's W
      // adjacent x-values are one contiguous 16W-byte run in the owning
      // rank's slab, so the transpose leaves as bulk-copy requests of whole
      // tile rows instead of 16-byte stores (NVLink to peers).
      if constexpr (MODE != COL_FWD) fft_line<L, E, 1, true, false>(v, t, tw, SmemBuf{xb, 0}, SyncAll{});
      __syncthreads();  // every exchange read is done before outputs overwrite the slot
      const bool inv_layout = (MODE != COL_FWD);
#pragma unroll
      for (int i = 0; i < E; ++i) slot[(comp * L + pos_last<L, E>(inv_layout, t, i)) * W + w] = v[0][i];
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
#else
      if constexpr (MODE != COL_FWD) fft_line<L, E, 1, true>(v, t, tw, SmemBuf{xb, 0}, SyncAll{});
      const bool inv_layout = (MODE != COL_FWD);
      const int rq = po->rows_per_rank;
      if (po->zs > 0) {  // z-blocked destination slabs
        const int zs = po->zs, msk = (1 << zs) - 1;
        const long long O = po->outer0 + o;
        const long long cbase = comp * po->comp_stride + x0 + w;
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int pos = pos_last<L, E>(inv_layout, t, i);
          const int q = pos / rq;
          const long long p = pos - q * rq;
          const long long b = po->blk_line ? p : O, u = po->blk_line ? O : p;
          const long long row = (((b >> zs) * po->bn + u) << zs) | (b & msk);
          po->dst[f][q][cbase + row * po->row_len] = v[0][i];
        }
      } else {
        const long long base = comp * po->comp_stride + (po->outer0 + o) * po->outer_stride + x0 + w;
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int pos = pos_last<L, E>(inv_layout, t, i);
          const int q = pos / rq;
          po->dst[f][q][base + (long long)(pos - q * rq) * po->line_stride] = v[0][i];
        }
      }
      __syncthreads();  // the slot's exchange reads are done before the next tile lands
#endif
    } else if (!parseval_only) {
      // (the explicit barrier below orders the inverse's last exchange reads)
      if constexpr (MODE != COL_FWD) fft_line<L, E, 1, true, false>(v, t, tw, SmemBuf{xb, 0}, SyncAll{});
      __syncthreads();  // every exchange read is done before outputs overwrite the slot
      const bool inv_layout = (MODE != COL_FWD);
#pragma unroll
      for (int i = 0; i < E; ++i) slot[(comp * L + pos_last<L, E>(inv_layout, t, i)) * W + w] = v[0][i];
      fence_proxy_async();
      __syncthreads();
      if (threadIdx.x == 0) {
        col3_store(f == 0 ? &tmA : &tmB, slot, x0, col3_outer(g, o));
        bulk_commit();
      }
    }  // parseval-only tiles: the projection's closing barrier released the slot
  }
  if (threadIdx.x == 0 || (PEER && FFTC_PEER_BULK)) bulk_wait0();  // stores have landed in global memory
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
