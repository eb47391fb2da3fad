// general.cuh -- the iteration for grids outside the fused transforms'
// lengths (any even axis length, reference geometry.py:37 / :93; the fused
// sweeps need powers of two 2..4096).
//
// Same algebra and device state as the fused sweeps (reference
// solvers.py:300-321 / :395-432, spectral_ops.py:120-128, the monitor of
// solvers.py:243-277), split into three pointwise kernels around cuFFT
// (library transforms, like cuBLAS for a plain GEMM):
//   k_gen_pro   prologue of sweep 1: the fields to transform, <j>, sum |Js|^2 chi
//   (cuFFT forward of A and, for EM-type schemes, B)
//   k_gen_gamma Gamma^ = k k^T / |k|^2 on every wave vector, Parseval residual,
//               the monitor in the last CTA (as the projection sweeps)
//   (cuFFT inverse of A)
//   k_gen_epi   epilogue of sweep 3: state update, <Q_raw> -> next delta
// Fields keep the reference (c, z, y, x) layout; every reduction is a fixed
// order tree (grid_reduce), so repeats are bit identical.
#pragma once
#include "sweeps.cuh"

namespace fftc {

template <int S>
__global__ void __launch_bounds__(256) k_gen_pro(Args a) {
  constexpr int NQ = Sweep1Traits<S>::NQ;
  if (a.st->stopped) return;
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  const long long total = (long long)a.d * a.N;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i / a.N);
    const long long p = i - (long long)c * a.N;
    const bool in1 = a.chi[p] != 0;
    const double2 dl = a.st->delta[c];
    const double2 q = a.X[0][i];
    if constexpr (S == BASIC) {
      const double2 j = cmul(sigma_at(a, in1), cadd(q, dl));  // j = sigma e (solvers.py:310-311)
      a.A[i] = j;
      acc_c<NQ>(acc, c, j);
    } else if constexpr (S == EM) {
      const double2 j = cmul(sigma_at(a, in1), cadd(q, dl));
      a.A[i] = cmul(in1 ? a.sm1 : a.sm2, q);  // r = (sigma - s0) e_raw (:303)
      a.B[i] = j;
      acc_c<NQ>(acc, c, j);
    } else {
      const double2 sv = in1 ? a.X[1][i] : czero();
      const double2 tv = (S == EM_SUB && in1) ? a.X[2][i] : czero();
      const AugFlux f = apply_A(a, in1, q, sv, tv);  // (:412)
      double2 jq, js;
      pinned_flux(a, in1, f.jq, f.js, dl, jq, js);
      acc_c<NQ>(acc, c, jq);
      if (in1) acc[NQ - 1] += cabs2(js);  // sum |Js|^2 chi (:429)
      if constexpr (S == BASIC_SUB) {
        a.A[i] = jq;
      } else {
        a.A[i] = csub(f.jq, cmul(a.s0, q));  // Rq = Jq_raw - s0 Q_raw (:398)
        a.B[i] = jq;
      }
    }
  }
  double tot[NQ];
  if (grid_reduce<NQ>(acc, tot, a) && threadIdx.x == 0) {
    for (int c = 0; c < a.d; ++c) a.st->jmean[c] = make_double2(tot[2 * c] * a.inv_n, tot[2 * c + 1] * a.inv_n);
    a.st->js2 = (NQ > 6) ? tot[NQ - 1] : 0.0;
  }
}

// MODE: MID_BASIC (A <- Gamma^ A, Parseval of it) or MID_EM (A <- (I - 2
// Gamma^) A, Parseval of Gamma^ B); spectra unnormalised (cuFFT forward)
template <int MODE>
__global__ void __launch_bounds__(256) k_gen_gamma(Args a) {
  if (!a.op_mode && a.st->stopped) return;
  double acc[1] = {0.0};
  const long long nxy = (long long)a.nx * a.ny;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < a.N; p += (long long)gridDim.x * blockDim.x) {
    const int z = (int)(p / nxy);
    const long long r = p - (long long)z * nxy;
    const int y = (int)(r / a.nx), x = (int)(r - (long long)y * a.nx);
    double k[3];
    k[0] = (double)wavenum(x, a.nx);
    k[1] = (double)wavenum(y, a.ny);
    k[2] = a.d == 3 ? (double)wavenum(z, a.nz) : 0.0;
    const double k2 = a.d == 3 ? k[0] * k[0] + k[1] * k[1] + k[2] * k[2] : k[0] * k[0] + k[1] * k[1];
    const double ik2 = (k2 != 0.0) ? inv_k2(k2) * a.gscale : 0.0;
    // field A
    {
      double2 F[3];
      for (int c = 0; c < a.d; ++c) F[c] = a.A[(size_t)c * a.N + p];
      double2 dot = cadd(cscale(F[0], k[0]), cscale(F[1], k[1]));  // kx F_x + ky F_y (+ kz F_z)
      if (a.d == 3) dot = cadd(dot, cscale(F[2], k[2]));
      dot = cscale(dot, ik2);
      for (int c = 0; c < a.d; ++c) {
        if constexpr (MODE == MID_BASIC) {
          const double2 g = cscale(dot, k[c]);
          acc[0] += cabs2(cscale(g, a.inv_n));  // Parseval on the 1/N-scaled mode
          // operator mode (fftc_gamma1): the inverse transform's 1/N here
          a.A[(size_t)c * a.N + p] = a.op_mode ? cscale(g, a.inv_n) : g;
        } else {
          a.A[(size_t)c * a.N + p] = csub(F[c], cscale(dot, 2.0 * k[c]));
        }
      }
    }
    if constexpr (MODE == MID_EM) {  // field B: Parseval only
      double2 F[3];
      for (int c = 0; c < a.d; ++c) F[c] = a.B[(size_t)c * a.N + p];
      double2 dot = cadd(cscale(F[0], k[0]), cscale(F[1], k[1]));
      if (a.d == 3) dot = cadd(dot, cscale(F[2], k[2]));
      dot = cscale(dot, ik2);
      for (int c = 0; c < a.d; ++c) acc[0] += cabs2(cscale(cscale(dot, k[c]), a.inv_n));
    }
  }
  double tot[1];
  if (grid_reduce<1>(acc, tot, a) && threadIdx.x == 0 && !a.op_mode) monitor_step(a, tot[0] / a.inv_n + a.st->js2);
}

template <int S>
__global__ void __launch_bounds__(256) k_gen_epi(Args a) {
  constexpr int NQ = 6;
  if (a.st->stopped) return;
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  const long long total = (long long)a.d * a.N;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i / a.N);
    const long long p = i - (long long)c * a.N;
    const bool in1 = a.chi[p] != 0;
    const double2 dl = a.st->delta[c];
    const double2 gq = cscale(a.A[i], a.inv_n);  // ifft normalisation 1/N
    double2 qn;
    if constexpr (S == BASIC) {
      qn = csub(cadd(a.X[0][i], dl), cmul(gq, a.inv_s0));  // e_raw <- (e_raw + delta) - g / s0 (:306)
    } else if constexpr (S == EM) {
      qn = cmul(cadd(a.two_s0_e0[c], gq), in1 ? a.inv_sum1 : a.inv_sum2);
    } else if constexpr (S == BASIC_SUB) {
      const double2 q = a.X[0][i];
      qn = csub(cadd(q, dl), cmul(gq, a.inv_s0));
      if (in1) {
        const double2 sv = a.X[1][i];
        const AugFlux f = apply_A(a, true, q, sv, czero());
        double2 jq, js;
        pinned_flux(a, true, f.jq, f.js, dl, jq, js);
        a.X[1][i] = csub(sv, cmul(js, a.inv_s0));
      }
    } else {
      const double2 wq = cadd(a.two_s0_e0[c], gq);
      double2 ws = czero(), wt = czero();
      if (in1) {
        const double2 q = a.X[0][i], sv = a.X[1][i], tv = a.X[2][i];
        const AugFlux f = apply_A(a, true, q, sv, tv);
        const double2 rs = csub(f.js, cmul(a.s0, sv));
        ws = make_double2(-rs.x, -rs.y);
        wt = csub(f.jt, cmul(a.s0, tv));
      }
      double2 sn, tn;
      em_sub_update(a, in1, wq, ws, wt, qn, sn, tn);
      if (in1) {
        a.X[1][i] = sn;
        a.X[2][i] = tn;
      }
    }
    a.X[0][i] = qn;
    acc_c<NQ>(acc, c, qn);
  }
  double tot[NQ];
  if (grid_reduce<NQ>(acc, tot, a) && threadIdx.x == 0) {
    for (int c = 0; c < a.d; ++c)
      a.st->delta[c] = csub(a.e0[c], make_double2(tot[2 * c] * a.inv_n, tot[2 * c + 1] * a.inv_n));
  }
}

}  // namespace fftc
