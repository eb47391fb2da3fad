// fft_engine.cuh -- register/shared-memory Stockham FFT for fp64 complex lines.
//
// Replaces the FFT arithmetic the reference gets from numpy's pocketfft
// (numpy.fft.fft2 / ifft2 called at reference spectral_ops.py:123,128).
// Design (B200, sm_100a):
//   * one 1-D transform of power-of-two length L is executed by T = L/E
//     threads, each holding E complex doubles per channel in registers;
//   * a thread may carry C channels (field components / fields) through the
//     same transform so that twiddles are shared and pointwise operators that
//     mix channels (the Gamma projection k k^T/|k|^2) stay in registers;
//   * stages are radix-E butterflies (E in {2,4,8,16}); between stages data
//     is exchanged through padded shared memory (pad one slot every E
//     entries) which makes every exchange bank-conflict free for E >= 8;
//   * Stockham auto-sort: the first stage reads positions t + b*T + r*L/R
//     and the last stage writes positions t + b*T + r*L/R, both natural
//     order, so loads/stores to HBM are coalesced and a forward transform
//     followed by the inverse of the reversed plan needs no exchange in
//     between (the fused Gamma projection sits exactly there);
//   * twiddles come from a per-length table exp(-2 pi i m / L) computed on
//     the host in long double; each butterfly loads log2(R) of them and
//     builds the rest with at most three complex products.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fftc {

// ----------------------------------------------------------------------------
// complex helpers (double2 = re, im)
// ----------------------------------------------------------------------------
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ double2 czero() { return make_double2(0.0, 0.0); }
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ double2 mul_mi(double2 a) {
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}
// twiddle product respecting direction: a * (INV ? conj(w) : w)
template <bool INV>
__device__ __forceinline__ double2 ctw(double2 a, double2 w) {
  return INV ? make_double2(a.x * w.x + a.y * w.y, a.y * w.x - a.x * w.y) : cmul(a, w);
}

constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x >> 1); }

// ----------------------------------------------------------------------------
// fixed-size DFTs in registers (natural-order in and out)
// forward: X_k = sum_n x_n exp(-2 pi i n k / R); inverse: conjugate kernel.
// ----------------------------------------------------------------------------
template <bool INV>
__device__ __forceinline__ void dft2(double2& a, double2& b) {
  double2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <bool INV>
__device__ __forceinline__ void dft4(double2& a0, double2& a1, double2& a2, double2& a3) {
  double2 s02 = cadd(a0, a2), d02 = csub(a0, a2);
  double2 s13 = cadd(a1, a3), d13 = mul_mi<INV>(csub(a1, a3));
  a0 = cadd(s02, s13);
  a2 = csub(s02, s13);
  a1 = cadd(d02, d13);
  a3 = csub(d02, d13);
}

// W_R^m multiply for the internal twiddles of radix 8/16 (compile-time m).
// cos/sin(2 pi m / 16) for m = 0..15
__device__ __forceinline__ constexpr double c16(int m) {
  // exact-to-double constants
  constexpr double C1 = 0.92387953251128675613;  // cos(pi/8)
  constexpr double S1 = 0.38268343236508977173;  // sin(pi/8)
  constexpr double H = 0.70710678118654752440;   // sqrt(2)/2
  const double tab[16] = {1.0, C1, H, S1, 0.0, -S1, -H, -C1, -1.0, -C1, -H, -S1, 0.0, S1, H, C1};
  return tab[m & 15];
}
__device__ __forceinline__ constexpr double s16(int m) { return c16(m + 12); }  // sin(x) = cos(x - pi/2)

template <bool INV, int M16>
__device__ __forceinline__ double2 tw16(double2 a) {
  // a * exp(-+ 2 pi i M16 / 16)
  constexpr int m = M16 & 15;
  if constexpr (m == 0) {
    return a;
  } else if constexpr (m == 4) {
    return mul_mi<INV>(a);
  } else if constexpr (m == 8) {
    return make_double2(-a.x, -a.y);
  } else if constexpr (m == 12) {
    return mul_mi<!INV>(a);
  } else {
    constexpr double c = c16(m);
    constexpr double s = INV ? s16(m) : -s16(m);  // w = c + i s
    return make_double2(a.x * c - a.y * s, a.x * s + a.y * c);
  }
}

template <bool INV>
__device__ __forceinline__ void dft8(double2* x) {
  // even / odd radix-4 then combine with W8^k = W16^(2k)
  double2 e0 = x[0], e1 = x[2], e2 = x[4], e3 = x[6];
  double2 o0 = x[1], o1 = x[3], o2 = x[5], o3 = x[7];
  dft4<INV>(e0, e1, e2, e3);
  dft4<INV>(o0, o1, o2, o3);
  o1 = tw16<INV, 2>(o1);
  o2 = tw16<INV, 4>(o2);
  o3 = tw16<INV, 6>(o3);
  x[0] = cadd(e0, o0); x[4] = csub(e0, o0);
  x[1] = cadd(e1, o1); x[5] = csub(e1, o1);
  x[2] = cadd(e2, o2); x[6] = csub(e2, o2);
  x[3] = cadd(e3, o3); x[7] = csub(e3, o3);
}

template <bool INV>
__device__ __forceinline__ void dft16(double2* x) {
  // n = 4 n1 + n2, k = k1 + 4 k2
  double2 y[16];
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) {
    double2 a0 = x[n2], a1 = x[4 + n2], a2 = x[8 + n2], a3 = x[12 + n2];
    dft4<INV>(a0, a1, a2, a3);
    y[n2 * 4 + 0] = a0; y[n2 * 4 + 1] = a1; y[n2 * 4 + 2] = a2; y[n2 * 4 + 3] = a3;
  }
  // twiddles W16^(n2 k1)
  y[1 * 4 + 1] = tw16<INV, 1>(y[1 * 4 + 1]);
  y[1 * 4 + 2] = tw16<INV, 2>(y[1 * 4 + 2]);
  y[1 * 4 + 3] = tw16<INV, 3>(y[1 * 4 + 3]);
  y[2 * 4 + 1] = tw16<INV, 2>(y[2 * 4 + 1]);
  y[2 * 4 + 2] = tw16<INV, 4>(y[2 * 4 + 2]);
  y[2 * 4 + 3] = tw16<INV, 6>(y[2 * 4 + 3]);
  y[3 * 4 + 1] = tw16<INV, 3>(y[3 * 4 + 1]);
  y[3 * 4 + 2] = tw16<INV, 6>(y[3 * 4 + 2]);
  y[3 * 4 + 3] = tw16<INV, 9>(y[3 * 4 + 3]);
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    double2 a0 = y[0 * 4 + k1], a1 = y[1 * 4 + k1], a2 = y[2 * 4 + k1], a3 = y[3 * 4 + k1];
    dft4<INV>(a0, a1, a2, a3);
    x[k1 + 0] = a0; x[k1 + 4] = a1; x[k1 + 8] = a2; x[k1 + 12] = a3;
  }
}

template <int R, bool INV>
__device__ __forceinline__ void dftR(double2* x) {
  if constexpr (R == 1) {
  } else if constexpr (R == 2) {
    dft2<INV>(x[0], x[1]);
  } else if constexpr (R == 4) {
    dft4<INV>(x[0], x[1], x[2], x[3]);
  } else if constexpr (R == 8) {
    dft8<INV>(x);
  } else {
    static_assert(R == 16, "radix must be 1,2,4,8,16");
    dft16<INV>(x);
  }
}

// ----------------------------------------------------------------------------
// the plan: radices per stage.  Forward: [E, 2^rem, E, E, ...]; the inverse
// plan is the reverse, so fwd-last == inv-first (register-aligned handoff).
// ----------------------------------------------------------------------------
template <int L, int E>
struct Plan {
  static_assert((L & (L - 1)) == 0 && L >= 2, "L must be a power of two");
  static_assert((E & (E - 1)) == 0 && E >= 2 && E <= 16 && E <= L, "bad E");
  static constexpr int T = L / E;
  static constexpr int LG = ilog2(L), EG = ilog2(E);
  static constexpr int Q = LG / EG, REM = LG % EG;
  static constexpr int NST = Q + (REM ? 1 : 0);
  static constexpr int PS = EG;                     // pad shift: one pad slot every E entries
  static constexpr int LP = L + (L >> PS);          // padded buffer length
  __host__ __device__ static constexpr int radix_fwd(int s) {
    return REM == 0 ? E : (s == 1 ? (1 << REM) : E);
  }
  __host__ __device__ static constexpr int radix(bool inv, int s) { return inv ? radix_fwd(NST - 1 - s) : radix_fwd(s); }
  __host__ __device__ static constexpr int ns(bool inv, int s) {  // product of radices before stage s
    int p = 1;
    for (int i = 0; i < s; ++i) p *= radix(inv, i);
    return p;
  }
  // natural-order position of register element i of thread t on entry (stage 0)
  __host__ __device__ static constexpr int R_first(bool inv) { return radix(inv, 0); }
  __host__ __device__ static constexpr int R_last(bool inv) { return radix(inv, NST - 1); }
};

template <int L, int E>
__device__ __forceinline__ int pos_first(bool inv, int t, int i) {
  using P = Plan<L, E>;
  const int R = P::R_first(inv);
  return t + (i / R) * P::T + (i % R) * (L / R);
}
template <int L, int E>
__device__ __forceinline__ int pos_last(bool inv, int t, int i) {
  using P = Plan<L, E>;
  const int R = P::R_last(inv);
  return t + (i / R) * P::T + (i % R) * (L / R);
}

template <int PS>
__device__ __forceinline__ int padpos(int p) { return p + (p >> PS); }

// Twiddle bases of one butterfly: w, w^2, w^4, w^8 of w = tw[m] (table
// loads).  Loaded one stage ahead -- before the exchange barrier that
// precedes the stage -- so the L1/L2 latency hides behind the exchange.
struct TwBase {
  double2 w1, w2, w4, w8;
};

// Twiddle tables: global (read-only path) or a shared-memory copy.
__device__ __forceinline__ double2 ld_tw(const double2* __restrict__ tw, int m) { return __ldg(&tw[m]); }
// Shared-memory copy of a table, swizzled so that any 8 consecutive
// multiples of a power-of-two stride land in 8 distinct 16-byte bank groups
// (a Stockham stage with Ns*R < L reads w^(k*L/(Ns*R)): strides 16..64 that
// would otherwise put a whole 8-lane LDS.128 phase in one bank group).
__host__ __device__ __forceinline__ int tw_swz(int m) { return (m & ~7) | ((m ^ (m >> 3) ^ (m >> 6) ^ (m >> 9)) & 7); }
struct SmemTw {
  const double2* p;  // table stored at tw_swz(m)
};
__device__ __forceinline__ double2 ld_tw(SmemTw tw, int m) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "r"((unsigned)__cvta_generic_to_shared(tw.p + tw_swz(m))));
  return v;
}

template <int R, class TW>
__device__ __forceinline__ TwBase load_twbase(TW tw, int m) {
  TwBase b;
  b.w1 = ld_tw(tw, m);
  if constexpr (R >= 4) b.w2 = ld_tw(tw, 2 * m);
  if constexpr (R >= 8) b.w4 = ld_tw(tw, 4 * m);
  if constexpr (R >= 16) b.w8 = ld_tw(tw, 8 * m);
  return b;
}

// Multiply element r of every channel by w^r (direction INV), r = 1..R-1,
// powers from the bases with at most three complex products each; each power
// is applied as soon as it is formed so few twiddles are live at once.
template <int C, int E, bool INV>
__device__ __forceinline__ void twmul(double2 (&v)[C][E], int idx, double2 w) {
#pragma unroll
  for (int c = 0; c < C; ++c) v[c][idx] = ctw<INV>(v[c][idx], w);
}

template <int R, int C, int E, bool INV>
__device__ __forceinline__ void apply_twiddles(double2 (&v)[C][E], int base, const TwBase& b) {
  const double2 w1 = b.w1;
  twmul<C, E, INV>(v, base + 1, w1);
  if constexpr (R >= 4) {
    const double2 w2 = b.w2;
    twmul<C, E, INV>(v, base + 2, w2);
    const double2 w3 = cmul(w1, w2);
    twmul<C, E, INV>(v, base + 3, w3);
    if constexpr (R >= 8) {
      const double2 w4 = b.w4;
      twmul<C, E, INV>(v, base + 4, w4);
      twmul<C, E, INV>(v, base + 5, cmul(w1, w4));
      twmul<C, E, INV>(v, base + 6, cmul(w2, w4));
      const double2 w7 = cmul(w3, w4);
      twmul<C, E, INV>(v, base + 7, w7);
      if constexpr (R >= 16) {
        const double2 w8 = b.w8;
        twmul<C, E, INV>(v, base + 8, w8);
        twmul<C, E, INV>(v, base + 9, cmul(w1, w8));
        twmul<C, E, INV>(v, base + 10, cmul(w2, w8));
        twmul<C, E, INV>(v, base + 11, cmul(w3, w8));
        twmul<C, E, INV>(v, base + 12, cmul(w4, w8));
        twmul<C, E, INV>(v, base + 13, cmul(cmul(w1, w4), w8));
        twmul<C, E, INV>(v, base + 14, cmul(cmul(w2, w4), w8));
        twmul<C, E, INV>(v, base + 15, cmul(w7, w8));
      }
    }
  }
}

// twiddle bases of every butterfly a thread owns in stage S
template <int L, int E, bool INV, int S>
struct StageTw {
  using P = Plan<L, E>;
  static constexpr int R = P::radix(INV, S);
  static constexpr int Ns = P::ns(INV, S);
  static constexpr int NB = (Ns > 1) ? E / R : 1;
  TwBase b[NB];
  template <class TW>
  __device__ __forceinline__ void load(int t, TW tw) {
    if constexpr (Ns > 1) {
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        const int j = t + k * P::T;
        b[k] = load_twbase<R>(tw, (j & (Ns - 1)) * (L / (Ns * R)));
      }
    }
  }
};

// One Stockham stage (compute only, registers in place).
template <int L, int E, int C, bool INV, int S>
__device__ __forceinline__ void stage_compute(double2 (&v)[C][E], const StageTw<L, E, INV, S>& tws) {
  using P = Plan<L, E>;
  constexpr int R = P::radix(INV, S);
  constexpr int Ns = P::ns(INV, S);
#pragma unroll
  for (int b = 0; b < E / R; ++b) {
    if constexpr (Ns > 1) apply_twiddles<R, C, E, INV>(v, b * R, tws.b[b]);
#pragma unroll
    for (int c = 0; c < C; ++c) dftR<R, INV>(&v[c][b * R]);
  }
}

// Exchange between stage S and S+1 through shared memory.  `buf(c)` is the
// padded buffer of channel c for this transform.  `bar` synchronises all
// threads sharing the buffers (normally __syncthreads).
template <int L, int E, int C, bool INV, int S, class Buf, class Bar, bool TAIL = true>
__device__ __forceinline__ void stage_exchange(double2 (&v)[C][E], int t, Buf buf, Bar bar) {
  using P = Plan<L, E>;
  constexpr int R = P::radix(INV, S);
  constexpr int Ns = P::ns(INV, S);
  constexpr int R2 = P::radix(INV, S + 1);
  constexpr int T = P::T;
  constexpr int PAD = 1 << P::PS;
  // When the stride between a butterfly's outputs (Ns) is a multiple of the
  // pad period, or the first stage writes a full pad period per butterfly,
  // every padded address is the butterfly base plus a compile-time offset.
  constexpr bool ST_CONST = (Ns % PAD == 0) || (Ns == 1 && R == PAD);
  constexpr int LD_STRIDE = L / R2;
  constexpr bool LD_CONST = (LD_STRIDE % PAD == 0);
#pragma unroll
  for (int b = 0; b < E / R; ++b) {
    const int j = t + b * T;
    const int base = (j / Ns) * Ns * R + (j & (Ns - 1));
    if constexpr (ST_CONST) {
      const int pb = padpos<P::PS>(base);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        constexpr int dummy = 0;
        (void)dummy;
        const int off = (Ns == 1) ? r : r * Ns + ((r * Ns) >> P::PS);
#pragma unroll
        for (int c = 0; c < C; ++c) buf(c)[pb + off] = v[c][b * R + r];
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c) buf(c)[padpos<P::PS>(base + r * Ns)] = v[c][b * R + r];
    }
  }
  bar();
#pragma unroll
  for (int b = 0; b < E / R2; ++b) {
    const int j = t + b * T;
    if constexpr (LD_CONST) {
      const int pj = padpos<P::PS>(j);
#pragma unroll
      for (int r = 0; r < R2; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c) v[c][b * R2 + r] = buf(c)[pj + r * LD_STRIDE + ((r * LD_STRIDE) >> P::PS)];
    } else {
#pragma unroll
      for (int r = 0; r < R2; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c) v[c][b * R2 + r] = buf(c)[padpos<P::PS>(j + r * LD_STRIDE)];
    }
  }
  if constexpr (TAIL) bar();
}

template <int L, int E, int C, bool INV, int S, bool TAIL, class Buf, class Bar, class TW>
__device__ __forceinline__ void run_from(double2 (&v)[C][E], int t, TW tw, Buf buf, Bar bar,
                                         const StageTw<L, E, INV, S>& tws) {
  using P = Plan<L, E>;
  stage_compute<L, E, C, INV, S>(v, tws);
  if constexpr (S + 1 < P::NST) {
    StageTw<L, E, INV, S + 1> nxt;
    nxt.load(t, tw);  // in flight during the exchange
    stage_exchange<L, E, C, INV, S, Buf, Bar, (TAIL || S + 2 < P::NST)>(v, t, buf, bar);
    run_from<L, E, C, INV, S + 1, TAIL>(v, t, tw, buf, bar, nxt);
  }
}

// Full length-L transform of C channels.  Input: element i of thread t sits
// at pos_first(INV,t,i); output: element i at pos_last(INV,t,i).
// TAIL = false drops the barrier after the last exchange's reads: only for
// callers that pass another barrier before anything writes the buffer again.
template <int L, int E, int C, bool INV, bool TAIL = true, class Buf, class Bar, class TW>
__device__ __forceinline__ void fft_line(double2 (&v)[C][E], int t, TW tw, Buf buf, Bar bar) {
  StageTw<L, E, INV, 0> first;  // stage 0 has Ns = 1: no twiddles
  run_from<L, E, C, INV, 0, TAIL>(v, t, tw, buf, bar, first);
}

// ----------------------------------------------------------------------------
// TMA bulk copy (global -> shared) completed on an mbarrier (sm_90+ PTX)
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 1/k2 for an integer-valued k2 >= 1 (|k|^2 of a wave vector): float seed
// plus two Newton steps in fp64, branch free (the IEEE division of the
// plain form carries a slow path per element); within 1 ulp of 1.0/k2.
__device__ __forceinline__ double inv_k2(double k2) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(k2));
  y = fma(y, fma(-k2, y, 1.0), y);
  y = fma(y, fma(-k2, y, 1.0), y);
  return y;
}

// signed integer wave number of index i on an n-point periodic grid
// (numpy.fft.fftfreq(n, d=1/n): 0..n/2-1, -n/2..-1)
// (written with an explicit unsigned half-length: nvcc 12.9 -O3 dropped the
// n/2 shift of the plain `i < n / 2` form in some instantiations)
__device__ __forceinline__ int wavenum(int i, int n) {
  const unsigned half = ((unsigned)n) >> 1;
  return ((unsigned)i >= half) ? i - n : i;
}

}  // namespace fftc
