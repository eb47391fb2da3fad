// ops.cu -- pointwise operators and deterministic reductions on device
// fields: the B200 side of the reference's public operator surface
// (fftcond/spectral_ops.py:96-278, fftcond/solvers.py:147-204).
//
// Fields are component-major complex128 (c, z, y, x) like VectorField.data
// (spectral_ops.py:58-70); an augmented field is three such fields (Q, S, T)
// (spectral_ops.py:141-173).  All kernels are HBM-streaming: one thread per
// voxel, all d components of that voxel, so every load/store is a coalesced
// 16-byte access and chi is read once per voxel.
//
// Reductions follow a fixed order (grid-stride partials over a fixed grid,
// warp-shuffle trees, one final CTA), so a result depends only on the
// inputs -- the reference's determinism requirement for its compensated
// sums (spectral_ops.py:33-55) -- though not bit-equal to math.fsum.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>

#include "../../include/fftcond_b200.h"
#include "host_common.h"

namespace fftc_ops {

struct c2 {
  double x, y;
};
__device__ __forceinline__ double2 mk(double x, double y) { return make_double2(x, y); }
__device__ __forceinline__ double2 add(double2 a, double2 b) { return mk(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 sub(double2 a, double2 b) { return mk(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 mul(double2 a, double2 b) { return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }

struct AugCoef {
  double2 p1, p2, p3;
  double2 tm1;    // t - 1
  double2 c;      // (t - 1)/(t + sigma0)       (invert_shifted_A)
  double2 scale;  // 1/(1 + sigma0)
};

// spectral_ops.py:215-278.  Operation order follows the reference so the
// results agree to the last bits in the common cases:
//   u  = chi ? p1 q + p2 s + p3 t : 0                   (_chi_aug_arrays :215-224)
//   CHI: (p1 u, p2 u, p3 u)                             (apply_chi_aug :227-237)
//   A:   ((t-1)(p1 u) + q, chi ? (t-1)(p2 u) + s : 0, ...) (apply_local_A :240-250)
//   INV: (sc (q - c (p1 u)), chi ? sc (s - c (p2 u)) : 0, ...) (invert_shifted_A :253-278)
template <int OP>
__global__ void __launch_bounds__(256) k_aug_apply(const uint8_t* __restrict__ chi, long long N, int d, AugCoef k,
                                                   const double2* __restrict__ Q, const double2* __restrict__ S,
                                                   const double2* __restrict__ T, double2* Qo, double2* So,
                                                   double2* To) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    const bool in1 = chi[i] != 0;
    for (int c = 0; c < d; ++c) {
      const long long o = (long long)c * N + i;
      const double2 q = Q[o], s = S[o], t = T[o];
      double2 u = add(add(mul(k.p1, q), mul(k.p2, s)), mul(k.p3, t));
      if (!in1) u = mk(0.0, 0.0);
      const double2 qo = mul(k.p1, u), so = mul(k.p2, u), to = mul(k.p3, u);
      double2 rq, rs, rt;
      if (OP == FFTC_AUG_CHI) {
        rq = qo;
        rs = so;
        rt = to;
      } else if (OP == FFTC_AUG_LOCAL_A) {
        rq = add(mul(k.tm1, qo), q);
        rs = in1 ? add(mul(k.tm1, so), s) : mk(0.0, 0.0);
        rt = in1 ? add(mul(k.tm1, to), t) : mk(0.0, 0.0);
      } else {
        rq = mul(k.scale, sub(q, mul(k.c, qo)));
        rs = in1 ? mul(k.scale, sub(s, mul(k.c, so))) : mk(0.0, 0.0);
        rt = in1 ? mul(k.scale, sub(t, mul(k.c, to))) : mk(0.0, 0.0);
      }
      Qo[o] = rq;
      So[o] = rs;
      To[o] = rt;
    }
  }
}

// j = sigma e with sigma = sigma1 on chi, 1 + 0i elsewhere (solvers.py:155, :286)
__global__ void __launch_bounds__(256) k_apply_sigma(const uint8_t* __restrict__ chi, long long N, int d, double2 s1,
                                                     const double2* __restrict__ e, double2* j) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    const double2 sg = chi[i] ? s1 : mk(1.0, 0.0);
    for (int c = 0; c < d; ++c) {
      const long long o = (long long)c * N + i;
      j[o] = mul(sg, e[o]);
    }
  }
}

// ---- deterministic reductions ------------------------------------------------
constexpr int RT = 256;       // threads per reduction CTA
constexpr int RGRID = 1024;   // fixed partial count (independent of the device)
constexpr int NQMAX = 6;

template <int NQ>
__device__ __forceinline__ void block_sum(double (&v)[NQ], double (&red)[RT / 32][NQMAX]) {
#pragma unroll
  for (int q = 0; q < NQ; ++q)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_down_sync(0xffffffffu, v[q], o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NQ; ++q) red[w][q] = v[q];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      double s = 0.0;
      for (int k = 0; k < RT / 32; ++k) s += red[k][q];
      v[q] = s;
    }
  }
}

// OP: FFTC_RED_SUM (NQ = 2d), FFTC_RED_DOT (2), FFTC_RED_NORM2 (1), FFTC_RED_OFF_SUPPORT (1)
template <int OP, int NQ>
__global__ void __launch_bounds__(RT) k_reduce(const uint8_t* __restrict__ chi, int mask, long long N, int d,
                                               const double2* __restrict__ a, const double2* __restrict__ b,
                                               double* partials) {
  __shared__ double red[RT / 32][NQMAX];
  double v[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) v[q] = 0.0;
  for (long long i = blockIdx.x * (long long)RT + threadIdx.x; i < N; i += (long long)gridDim.x * RT) {
    const bool in1 = chi ? chi[i] != 0 : true;
    if (OP == FFTC_RED_OFF_SUPPORT) {
      if (in1) continue;
      bool nz = false;
      for (int c = 0; c < d; ++c) {
        const double2 x = a[(long long)c * N + i];
        nz |= (x.x != 0.0) || (x.y != 0.0);
        if (b) {
          const double2 y = b[(long long)c * N + i];
          nz |= (y.x != 0.0) || (y.y != 0.0);
        }
      }
      v[0] += nz ? 1.0 : 0.0;
      continue;
    }
    if (mask == FFTC_MASK_CHI && !in1) continue;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      if (c >= d) break;
      const long long o = (long long)c * N + i;
      const double2 x = a[o];
      if (OP == FFTC_RED_SUM) {
        if (2 * c + 1 < NQ) {
          v[2 * c] += x.x;
          v[2 * c + 1] += x.y;
        }
      } else if (OP == FFTC_RED_DOT) {
        const double2 y = b[o];
        v[0] += x.x * y.x + x.y * y.y;  // conj(a) b
        if (NQ > 1) v[NQ - 1] += x.x * y.y - x.y * y.x;
      } else {
        v[0] += x.x * x.x + x.y * x.y;
      }
    }
  }
  block_sum<NQ>(v, red);
  if (threadIdx.x == 0)
#pragma unroll
    for (int q = 0; q < NQ; ++q) partials[(size_t)blockIdx.x * NQ + q] = v[q];
}

template <int NQ>
__global__ void __launch_bounds__(RT) k_reduce_final(const double* __restrict__ partials, int np, double* out) {
  __shared__ double red[RT / 32][NQMAX];
  double v[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) v[q] = 0.0;
  for (int b = threadIdx.x; b < np; b += RT)
#pragma unroll
    for (int q = 0; q < NQ; ++q) v[q] += partials[(size_t)b * NQ + q];
  block_sum<NQ>(v, red);
  if (threadIdx.x == 0)
#pragma unroll
    for (int q = 0; q < NQ; ++q) out[q] = v[q];
}

// ---- host helpers ----------------------------------------------------------------
struct Geo {
  int d;
  long long N;
};

int geo(const fftc_problem* pb, Geo& g, bool need_chi) {
  if (!pb || (pb->d != 2 && pb->d != 3)) {
    fftc::set_last_error("d must be 2 or 3");
    return 2;
  }
  g.d = pb->d;
  const long long nz = pb->d == 3 ? pb->n[2] : 1;
  if (pb->n[0] < 1 || pb->n[1] < 1 || nz < 1) {
    fftc::set_last_error("grid dimensions must be positive");
    return 2;
  }
  g.N = pb->n[0] * pb->n[1] * nz;
  if (need_chi && !pb->chi) {
    fftc::set_last_error("chi (device phase map) is required");
    return 2;
  }
  return 0;
}

int grid_for(long long N) {
  const long long want = (N + 255) / 256;
  const long long cap = (long long)fftc::device_sm_count() * 8;
  return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fftc::set_last_error(std::string(what) + ": " + cudaGetErrorString(e));
    return 1;
  }
  return 0;
}

inline double2 cd(const double* p) { return make_double2(p[0], p[1]); }
inline double2 hmul(double2 a, double2 b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
inline double2 hdiv(double2 a, double2 b) {
  // complex division the way CPython does it (Smith's algorithm), so the
  // shared coefficients match complex arithmetic on the host
  const double abs_br = b.x < 0 ? -b.x : b.x, abs_bi = b.y < 0 ? -b.y : b.y;
  if (abs_br >= abs_bi) {
    if (abs_br == 0.0) return make_double2(a.x / 0.0, a.y / 0.0);
    const double ratio = b.y / b.x, den = b.x + b.y * ratio;
    return make_double2((a.x + a.y * ratio) / den, (a.y - a.x * ratio) / den);
  }
  const double ratio = b.x / b.y, den = b.x * ratio + b.y;
  return make_double2((a.x * ratio + a.y) / den, (a.y * ratio - a.x) / den);
}

}  // namespace fftc_ops

using namespace fftc_ops;

extern "C" {

int fftc_aug_apply(const fftc_problem* pb, int32_t op, const double* coef, const void* Q, const void* S, const void* T,
                   void* Qo, void* So, void* To, void* stream) {
  fftc::clear_last_error();
  Geo g;
  if (int rc = geo(pb, g, true)) return rc;
  if (!coef || !Q || !S || !T || !Qo || !So || !To) {
    fftc::set_last_error("null argument");
    return 2;
  }
  AugCoef k;
  k.p1 = cd(coef + 0);
  k.p2 = cd(coef + 2);
  k.p3 = cd(coef + 4);
  const double2 t = cd(coef + 6), s0 = cd(coef + 8);
  k.tm1 = make_double2(t.x - 1.0, t.y);
  k.c = hdiv(k.tm1, make_double2(t.x + s0.x, t.y + s0.y));
  k.scale = hdiv(make_double2(1.0, 0.0), make_double2(1.0 + s0.x, s0.y));
  const int grid = grid_for(g.N);
  cudaStream_t s = (cudaStream_t)stream;
  auto args = [&](auto kern) {
    kern<<<grid, 256, 0, s>>>(pb->chi, g.N, g.d, k, (const double2*)Q, (const double2*)S, (const double2*)T,
                              (double2*)Qo, (double2*)So, (double2*)To);
  };
  switch (op) {
    case FFTC_AUG_CHI: args(k_aug_apply<FFTC_AUG_CHI>); break;
    case FFTC_AUG_LOCAL_A: args(k_aug_apply<FFTC_AUG_LOCAL_A>); break;
    case FFTC_AUG_INV_SHIFTED: args(k_aug_apply<FFTC_AUG_INV_SHIFTED>); break;
    default:
      fftc::set_last_error("bad augmented operator code");
      return 2;
  }
  fftc::add_launches(1);
  return check_launch("fftc_aug_apply");
}

int fftc_apply_sigma(const fftc_problem* pb, const double* sigma1, const void* e, void* j, void* stream) {
  fftc::clear_last_error();
  Geo g;
  if (int rc = geo(pb, g, true)) return rc;
  if (!sigma1 || !e || !j) {
    fftc::set_last_error("null argument");
    return 2;
  }
  k_apply_sigma<<<grid_for(g.N), 256, 0, (cudaStream_t)stream>>>(pb->chi, g.N, g.d, cd(sigma1), (const double2*)e,
                                                                 (double2*)j);
  fftc::add_launches(1);
  return check_launch("fftc_apply_sigma");
}

int fftc_reduce(const fftc_problem* pb, int32_t op, int32_t mask, const void* a, const void* b, double* out,
                void* stream) {
  fftc::clear_last_error();
  Geo g;
  const bool need_chi = (mask == FFTC_MASK_CHI) || (op == FFTC_RED_OFF_SUPPORT);
  if (int rc = geo(pb, g, need_chi)) return rc;
  if (!a || !out || (op == FFTC_RED_DOT && !b) || (mask != FFTC_MASK_NONE && mask != FFTC_MASK_CHI)) {
    fftc::set_last_error("null or invalid argument");
    return 2;
  }
  int nq;
  switch (op) {
    case FFTC_RED_SUM: nq = 2 * g.d; break;
    case FFTC_RED_DOT: nq = 2; break;
    case FFTC_RED_NORM2:
    case FFTC_RED_OFF_SUPPORT: nq = 1; break;
    default:
      fftc::set_last_error("bad reduction code");
      return 2;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const long long want = (g.N + RT - 1) / RT;
  const int grid = (int)(want < RGRID ? (want > 0 ? want : 1) : RGRID);
  double* ws = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&ws, sizeof(double) * ((size_t)grid * NQMAX + NQMAX), s);
  if (e != cudaSuccess) {
    fftc::set_last_error(std::string("fftc_reduce workspace: ") + cudaGetErrorString(e));
    return 1;
  }
  double* fin = ws + (size_t)grid * NQMAX;
  const uint8_t* chi = need_chi ? pb->chi : nullptr;
  const double2* A = (const double2*)a;
  const double2* B = (const double2*)b;
  switch (op) {
    case FFTC_RED_SUM:
      if (g.d == 2) {
        k_reduce<FFTC_RED_SUM, 4><<<grid, RT, 0, s>>>(chi, mask, g.N, g.d, A, B, ws);
        k_reduce_final<4><<<1, RT, 0, s>>>(ws, grid, fin);
      } else {
        k_reduce<FFTC_RED_SUM, 6><<<grid, RT, 0, s>>>(chi, mask, g.N, g.d, A, B, ws);
        k_reduce_final<6><<<1, RT, 0, s>>>(ws, grid, fin);
      }
      break;
    case FFTC_RED_DOT:
      k_reduce<FFTC_RED_DOT, 2><<<grid, RT, 0, s>>>(chi, mask, g.N, g.d, A, B, ws);
      k_reduce_final<2><<<1, RT, 0, s>>>(ws, grid, fin);
      break;
    case FFTC_RED_NORM2:
      k_reduce<FFTC_RED_NORM2, 1><<<grid, RT, 0, s>>>(chi, mask, g.N, g.d, A, B, ws);
      k_reduce_final<1><<<1, RT, 0, s>>>(ws, grid, fin);
      break;
    default:
      k_reduce<FFTC_RED_OFF_SUPPORT, 1><<<grid, RT, 0, s>>>(chi, mask, g.N, g.d, A, B, ws);
      k_reduce_final<1><<<1, RT, 0, s>>>(ws, grid, fin);
      break;
  }
  fftc::add_launches(2);
  int rc = check_launch("fftc_reduce");
  double host[NQMAX];
  if (!rc) {
    e = cudaMemcpyAsync(host, fin, sizeof(double) * nq, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      fftc::set_last_error(std::string("fftc_reduce: ") + cudaGetErrorString(e));
      rc = 1;
    }
  }
  cudaFreeAsync(ws, s);
  if (!rc) memcpy(out, host, sizeof(double) * nq);
  return rc;
}

}  // extern "C"
