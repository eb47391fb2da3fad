// abi.cu -- C-ABI entry points and the host driver of the iteration.
//
// fftc_solve() replaces the reference loops _solve_h / _solve_aug
// (reference solvers.py:280-331, :366-443).  Per iteration it launches the
// fused sweeps of sweeps.cuh; the stopping monitor runs on the device, so
// the host only synchronises once per chunk of iterations to collect the
// history ring and the stop flag.
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/fftcond_b200.h"
#include "host_common.h"
#include "kernel_table.h"
#include "sweeps.cuh"
#include "general.cuh"

#include <cufft.h>

using namespace fftc;

namespace {

thread_local std::string g_err;
std::atomic<long long> g_launches{0};

struct Registry {
  std::mutex mu;
  bool filled = false;
  LTable tab[MAX_LG + 1];
  const double2* tw[MAX_LG + 1] = {};  // device twiddle tables per length
  int num_sms = 0;
  int device = -1;
};
Registry& reg() {
  static Registry r;
  return r;
}

#define CK(expr)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (expr);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      g_err = std::string(#expr) + ": " + cudaGetErrorString(e_);                     \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

int lg2_exact(long long n) {
  if (n < 2 || (n & (n - 1))) return -1;
  int lg = 0;
  while ((1LL << lg) < n) ++lg;
  return lg <= MAX_LG ? lg : -1;
}

// an axis the solve accepts: even and >= 2, as the reference's PhaseMap
bool even_axis(long long n) { return n >= 2 && n % 2 == 0 && n <= (1LL << 30); }
// grids the fused sweeps do not cover go through general.cuh + cuFFT
bool general_grid(int d, long long nx, long long ny, long long nz) {
  if (const char* e = getenv("FFTC_GENERAL"))
    if (atoi(e) == 1) return true;
  return lg2_exact(nx) < 0 || lg2_exact(ny) < 0 || (d == 3 && lg2_exact(nz) < 0);
}

// exp(-2 pi i m / L), m = 0..L-1, in long double then rounded
std::vector<double2> make_twiddles(int L) {
  std::vector<double2> h(L);
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int m = 0; m < L; ++m) {
    // reduce by symmetry to keep the argument small
    long double ang = 2.0L * pi * (long double)m / (long double)L;
    h[m].x = (double)cosl(ang);
    h[m].y = (double)(-sinl(ang));
  }
  // exact values at the quadrant points
  h[0] = make_double2(1.0, 0.0);
  if (L % 4 == 0) {
    h[L / 4] = make_double2(0.0, -1.0);
    h[3 * L / 4] = make_double2(0.0, 1.0);
  }
  if (L % 2 == 0) h[L / 2] = make_double2(-1.0, 0.0);
  return h;
}

int ensure_registry() {
  Registry& r = reg();
  std::lock_guard<std::mutex> lk(r.mu);
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (r.filled && r.device == dev) return 0;
  fftc_fill_table_1(r.tab[1]);
  fftc_fill_table_2(r.tab[2]);
  fftc_fill_table_3(r.tab[3]);
  fftc_fill_table_4(r.tab[4]);
  fftc_fill_table_5(r.tab[5]);
  fftc_fill_table_6(r.tab[6]);
  fftc_fill_table_7(r.tab[7]);
  fftc_fill_table_8(r.tab[8]);
  fftc_fill_table_9(r.tab[9]);
  fftc_fill_table_10(r.tab[10]);
  fftc_fill_table_11(r.tab[11]);
  fftc_fill_table_12(r.tab[12]);
  CK(cudaDeviceGetAttribute(&r.num_sms, cudaDevAttrMultiProcessorCount, dev));
  {
    // workspaces come from the stream-ordered pool; keep freed blocks cached
    // so repeated solves do not map/unmap hundreds of MB per call
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
  }
  for (int lg = 1; lg <= MAX_LG; ++lg) {
    LTable& t = r.tab[lg];
    KInfo* all[4 + 4 + 3 + KC_COUNT + 2];  // NOLINT
    int n = 0;
    all[n++] = &t.row_fwd;
    all[n++] = &t.row_inv;
    all[n++] = &t.s1l[0];
    all[n++] = &t.s1l[1];
    all[n++] = &t.s3l;
    for (int s = 0; s < 4; ++s) all[n++] = &t.s1[s];
    for (int s = 0; s < 4; ++s) all[n++] = &t.s3[s];
    for (int c = 0; c < KC_COUNT; ++c) all[n++] = &t.col[c];
    for (int i = 0; i < n; ++i) {
      KInfo* k = all[i];
      if (!k->fn) continue;  // variant not instantiated for this length
      if (k->smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, k->smem);
        if (e != cudaSuccess) {  // too large for this device: mark unusable
          cudaGetLastError();
          k->max_active = 0;
          continue;
        }
      }
      int nb = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k->fn, k->threads, k->smem) != cudaSuccess) {
        cudaGetLastError();  // e.g. a configuration this device cannot run: leave it unusable
        nb = 0;
      }
      k->max_active = nb;
    }
    if (!r.tw[lg]) {
      std::vector<double2> h = make_twiddles(1 << lg);
      double2* d = nullptr;
      CK(cudaMalloc(&d, sizeof(double2) * h.size()));
      CK(cudaMemcpy(d, h.data(), sizeof(double2) * h.size(), cudaMemcpyHostToDevice));
      r.tw[lg] = d;
    }
  }
  r.device = dev;
  r.filled = true;
  return 0;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
    cudaGetLastError();
  });
  return fn;
}

// 4-D map over a (d, ny, nx) complex128 field seen as doubles
// {2nx, rows, ny/rows, d}: a box {2, rows, ny/rows, 2} is one whole column
// (both components, all ny rows, 16 B per row) in a single TMA operation.
bool make_field_map(CUtensorMap* tm, void* base, long long nx, long long ny, int d, int rows) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc || ny % rows) return false;
  cuuint64_t dims[4] = {(cuuint64_t)(2 * nx), (cuuint64_t)rows, (cuuint64_t)(ny / rows), (cuuint64_t)d};
  cuuint64_t strides[3] = {(cuuint64_t)(nx * 16), (cuuint64_t)(nx * 16 * rows), (cuuint64_t)(nx * ny * 16)};
  cuuint32_t box[4] = {2, (cuuint32_t)rows, (cuuint32_t)(ny / rows), 2};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS && getenv("FFTC_VERBOSE")) fprintf(stderr, "[fftc] cuTensorMapEncodeTiled failed: %d\n", (int)r);
  return r == CUDA_SUCCESS;
}

// 5-D map for the 3-D column passes: lines of length L at element stride
// line_stride, nouter of them at outer_stride, three components at
// comp_stride; a box is W adjacent x-columns of all three components
// {2W doubles, 256 rows, L/256 blocks, 1, 3} (cols3_lg.cuh).
// swz > 0: the TMA swizzle whose span is one box row (16 W bytes), cols3_lg.cuh
CUtensorMapSwizzle col3_swizzle(int swz) {
  return swz == 8 ? CU_TENSOR_MAP_SWIZZLE_128B
                  : (swz == 4 ? CU_TENSOR_MAP_SWIZZLE_64B : (swz == 2 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE));
}
bool make_line_map(CUtensorMap* tm, void* base, long long nx, long long L, int W, long long line_stride,
                   long long nouter, long long outer_stride, long long comp_stride, int swz, int ncb = 3) {
  EncodeTiledFn enc = encode_tiled();
  const long long rows = L < 256 ? L : 256;
  if (!enc || L % rows || nx % W) return false;
  cuuint64_t dims[5] = {(cuuint64_t)(2 * nx), (cuuint64_t)rows, (cuuint64_t)(L / rows), (cuuint64_t)nouter, 3};
  cuuint64_t strides[4] = {(cuuint64_t)(line_stride * 16), (cuuint64_t)(line_stride * 16 * rows),
                           (cuuint64_t)(outer_stride * 16), (cuuint64_t)(comp_stride * 16)};
  cuuint32_t box[5] = {(cuuint32_t)(2 * W), (cuuint32_t)rows, (cuuint32_t)(L / rows), 1, (cuuint32_t)ncb};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   col3_swizzle(swz), CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS && getenv("FFTC_VERBOSE")) fprintf(stderr, "[fftc] 5-D tensor map failed: %d\n", (int)r);
  return r == CUDA_SUCCESS;
}

// 5-D maps over a work field in the z-blocked layout (Args::zbs, ZB = 2^zbs
// z-planes of a y-row adjacent), box = W x-columns x one whole line x 3
// components landing as [c][pos][w] like make_line_map:
//   z lines (axis 2, outer y): {2nx, ZB (zl), nz/ZB (zh), ny, 3}
//   y lines (axis 1, outer z): {2nx, BY, (ny/BY)*(nz/ZB), ZB (zl), 3} -- the
//     y-block and zh dimensions fold into one because the zh step is exactly
//     ny/BY y-blocks; outer z sits at {(z >> zbs) * ny/BY, z & (ZB-1)}.
bool make_zblk_map(CUtensorMap* tm, void* base, long long nx, long long ny, long long nz, int W, int axis, int zbs,
                   int swz, int ncb = 3) {
  EncodeTiledFn enc = encode_tiled();
  const long long ZB = 1LL << zbs, N = nx * ny * nz;
  if (!enc || nx % W || nz % ZB) return false;
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5];
  if (axis == 2) {
    if (ZB > 256 || nz / ZB > 256) return false;
    const cuuint64_t d5[5] = {(cuuint64_t)(2 * nx), (cuuint64_t)ZB, (cuuint64_t)(nz / ZB), (cuuint64_t)ny, 3};
    const cuuint64_t s4[4] = {(cuuint64_t)(nx * 16), (cuuint64_t)(ny * ZB * nx * 16), (cuuint64_t)(ZB * nx * 16),
                              (cuuint64_t)(N * 16)};
    const cuuint32_t b5[5] = {(cuuint32_t)(2 * W), (cuuint32_t)ZB, (cuuint32_t)(nz / ZB), 1, (cuuint32_t)ncb};
    memcpy(dims, d5, sizeof(dims));
    memcpy(strides, s4, sizeof(strides));
    memcpy(box, b5, sizeof(box));
  } else {
    const long long BY = ny < 256 ? ny : 256;
    if (ny % BY) return false;
    const cuuint64_t d5[5] = {(cuuint64_t)(2 * nx), (cuuint64_t)BY, (cuuint64_t)((ny / BY) * (nz / ZB)), (cuuint64_t)ZB,
                              3};
    const cuuint64_t s4[4] = {(cuuint64_t)(ZB * nx * 16), (cuuint64_t)(BY * ZB * nx * 16), (cuuint64_t)(nx * 16),
                              (cuuint64_t)(N * 16)};
    const cuuint32_t b5[5] = {(cuuint32_t)(2 * W), (cuuint32_t)BY, (cuuint32_t)(ny / BY), 1, (cuuint32_t)ncb};
    memcpy(dims, d5, sizeof(dims));
    memcpy(strides, s4, sizeof(strides));
    memcpy(box, b5, sizeof(box));
  }
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   col3_swizzle(swz), CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS && getenv("FFTC_VERBOSE")) fprintf(stderr, "[fftc] z-blocked tensor map failed: %d\n", (int)r);
  return r == CUDA_SUCCESS;
}

// one TMA 3-D column pass: tiles of W x-columns x `nouter` outer lines,
// fields A (and B when given), all three components per tile
struct Col3Pass {
  const KInfo* k = nullptr;
  Line3 g{};
  CUtensorMap mA, mB;
  long long tiles = 0;
  bool ok = false;
};
bool col3_pass(Col3Pass& p, const KInfo& k, const Args& a, void* A, void* B, long long L, long long line_stride,
               long long nouter, long long outer_stride, long long comp_stride, int nfields, int axis, int o0, int on) {
  p.ok = false;
  p.g = Line3{};
  const char* sel = getenv("FFTC_TMA_COLS3");  // "0": the strip kernels (k_col), for comparison
  if (!k.fn || k.max_active <= 0 || (sel && atoi(sel) == 0)) return false;
  const int W = k.tile_w ? k.tile_w : col3_tile_w(L), ncb = k.tile_nc ? k.tile_nc : 3;
  if (a.nx % W) return false;
  if (!make_line_map(&p.mA, A, a.nx, L, W, line_stride, nouter, outer_stride, comp_stride, k.swz, ncb)) return false;
  if (!make_line_map(&p.mB, B ? B : A, a.nx, L, W, line_stride, nouter, outer_stride, comp_stride, k.swz, ncb))
    return false;
  p.k = &k;
  p.g.nouter = (int)nouter;
  p.g.o0 = o0;
  p.g.on = on;
  p.g.nfields = nfields;
  p.g.axis = axis;
  p.tiles = nouter * (a.nx / W) * nfields * (3 / ncb);
  p.ok = true;
  return true;
}

// the same pass over work fields in the z-blocked layout (monolithic 3-D solve)
bool col3_pass_zblk(Col3Pass& p, const KInfo& k, const Args& a, void* A, void* B, int axis, int zbs, int nfields) {
  p.ok = false;
  p.g = Line3{};
  const char* sel = getenv("FFTC_TMA_COLS3");
  if (!k.fn || k.max_active <= 0 || (sel && atoi(sel) == 0)) return false;
  const long long nx = a.nx, ny = a.ny, nz = a.nz;
  const long long L = axis == 2 ? nz : ny;
  const int W = k.tile_w ? k.tile_w : col3_tile_w(L), ncb = k.tile_nc ? k.tile_nc : 3;
  if (nx % W) return false;
  if (!make_zblk_map(&p.mA, A, nx, ny, nz, W, axis, zbs, k.swz, ncb)) return false;
  if (!make_zblk_map(&p.mB, B ? B : A, nx, ny, nz, W, axis, zbs, k.swz, ncb)) return false;
  p.k = &k;
  p.g.nouter = (int)(axis == 2 ? ny : nz);
  p.g.o0 = 0;
  p.g.on = (int)(axis == 2 ? ny : nz);
  p.g.nfields = nfields;
  p.g.axis = axis;
  p.g.obs = axis == 1 ? zbs : 0;
  p.g.om = axis == 1 ? (int)(ny / (ny < 256 ? ny : 256)) : 0;
  p.tiles = (long long)p.g.nouter * (nx / W) * nfields * (3 / ncb);
  p.ok = true;
  return true;
}

// z-block shift for the monolithic 3-D solve's work fields.  A y-line then
// spans ny*ZB*nx*16 B and a z-line nz/ZB blocks, one 2 MB page each; ZB
// balances the two page counts (ZB^2 = nz * 2^17 / (nx*ny)): 16 at 512^3 and
// 1024^3.  Measured at 1024^3 basic (scripts/kernels_3d.py): ZB = 1 (the
// reference layout) 174 ms/iteration, z pass 94 ms; ZB = 8/16/32/64 142 /
// 130 / 140 / 146 ms.  FFTC_ZBLOCK=<shift> overrides, 0 keeps the reference
// layout.
thread_local int g_last_zbs = 0;
int zblock_shift(long long nx, long long ny, long long nz) {
  int s = (int)std::floor(0.5 * std::log2((double)nz * 131072.0 / ((double)nx * (double)ny)) + 0.5);
  s = std::max(1, std::min(s, 6));
  if (const char* e = getenv("FFTC_ZBLOCK")) s = atoi(e);
  while (s > 0 && (1LL << s) > nz) --s;
  return s < 0 ? 0 : s;
}

double2 C2(const double* p) { return make_double2(p[0], p[1]); }
double2 hmul(double2 a, double2 b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
double2 hadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
double2 hsub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
double2 hinv(double2 a) {  // 1 / a (Smith)
  if (fabs(a.x) >= fabs(a.y)) {
    double r = a.y / a.x, den = a.x + a.y * r;
    return make_double2(1.0 / den, -r / den);
  }
  double r = a.x / a.y, den = a.x * r + a.y;
  return make_double2(r / den, -1.0 / den);
}
double2 hdiv(double2 a, double2 b) {
  if (fabs(b.x) >= fabs(b.y)) {
    double r = b.y / b.x, den = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / den, (a.y - a.x * r) / den);
  }
  double r = b.x / b.y, den = b.x * r + b.y;
  return make_double2((a.x * r + a.y) / den, (a.y * r - a.x) / den);
}

// Scalars of one solve (host side, mirroring the reference expressions:
// solvers.py:286-290, :369-392); the grid fields are filled by the caller.
void fill_scalars(Args& a, const fftc_params* pr, int d, long long N) {
  const double2 one = make_double2(1.0, 0.0);
  a.sigma1 = C2(pr->sigma1);
  a.s0 = C2(pr->sigma0);
  double e0sq = 0.0;
  for (int c = 0; c < 3; ++c) {
    a.e0[c] = c < d ? C2(pr->e0[c]) : make_double2(0, 0);
    e0sq += a.e0[c].x * a.e0[c].x + a.e0[c].y * a.e0[c].y;
  }
  a.e0sq = e0sq;
  a.tol = pr->tol;
  a.inv_n = 1.0 / (double)N;
  a.gscale = pr->gamma1_scale;
  a.max_iters = pr->max_iters;
  a.inv_s0 = hinv(a.s0);
  a.sum1 = hadd(a.sigma1, a.s0);
  a.sum2 = hadd(one, a.s0);
  a.inv_sum1 = hinv(a.sum1);
  a.inv_sum2 = hinv(a.sum2);
  a.sm1 = hsub(a.sigma1, a.s0);
  a.sm2 = hsub(one, a.s0);
  const double2 two_s0 = make_double2(2.0 * a.s0.x, 2.0 * a.s0.y);
  for (int c = 0; c < 3; ++c) a.two_s0_e0[c] = hmul(two_s0, a.e0[c]);
  const double2 t = C2(pr->t);
  a.p1 = C2(pr->p1);
  a.p2 = C2(pr->p2);
  a.p3 = C2(pr->p3);
  const double2 tm1 = hsub(t, one);
  a.tm1p1 = hmul(tm1, a.p1);
  a.tm1p2 = hmul(tm1, a.p2);
  a.tm1p3 = hmul(tm1, a.p3);
  a.cq = hmul(a.p1, a.tm1p1);
  a.cs = hmul(a.p2, a.tm1p1);
  a.sinv = hdiv(one, hadd(one, a.s0));            // inv_scale = 1/(1+s0)   (solvers.py:388)
  const double2 cinv = hdiv(tm1, hadd(t, a.s0));  // inv_c = (t-1)/(t+s0)  (solvers.py:389)
  a.cinv_p1 = hmul(cinv, a.p1);
  a.cinv_p2 = hmul(cinv, a.p2);
  a.cinv_p3 = hmul(cinv, a.p3);
}

// ---- optional per-kernel timing (fftc_profile): event pairs per launch ----
enum KindId { K_SWEEP1 = 0, K_MID, K_SWEEP3, K_YFWD, K_YINV, K_INIT, K_FINAL, K_OP, K_PARSEVAL, K_NKIND };
const char* kKindName[K_NKIND] = {"sweep1_rows_fwd", "sweep2_cols_gamma", "sweep3_rows_inv", "y_fwd_3d",
                                  "y_inv_3d", "init", "finalize", "operator", "z_parseval_3d"};
struct KindStat {
  long long launches = 0;
  double ms = 0.0;
};
std::mutex g_prof_mu;
bool g_profile = false;
KindStat g_stats[K_NKIND];

bool debug_sync() {
  static const bool on = getenv("FFTC_DEBUG_SYNC") != nullptr;
  return on;
}

struct Launcher {
  cudaStream_t s;
  int num_sms;
  long long count = 0;
  bool prof = false;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  std::vector<cudaEvent_t> pool;
  Launcher(cudaStream_t st, int sms) : s(st), num_sms(sms) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    prof = g_profile;
  }
  ~Launcher() {
    harvest();
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
  }
  cudaEvent_t ev() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  // call only after the stream has been synchronised
  void harvest() {
    if (pending.empty()) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto& p : pending) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, p.second.first, p.second.second) == cudaSuccess) {
        g_stats[p.first].launches += 1;
        g_stats[p.first].ms += ms;
      }
      pool.push_back(p.second.first);
      pool.push_back(p.second.second);
    }
    pending.clear();
  }
  int raw(const void* fn, unsigned grid, int threads, int smem, void** args, int kind) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (prof) {
      e0 = ev();
      e1 = ev();
      cudaEventRecord(e0, s);
    }
    CK(cudaLaunchKernel(fn, dim3(grid), dim3(threads), args, (size_t)smem, s));
    if (debug_sync()) {  // FFTC_DEBUG_SYNC=1: locate a faulting kernel
      cudaError_t e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) {
        g_err = std::string("kernel kind ") + kKindName[kind] + " grid " + std::to_string(grid) + " block " +
                std::to_string(threads) + " smem " + std::to_string(smem) + ": " + cudaGetErrorString(e);
        return 1;
      }
    }
    if (prof) {
      cudaEventRecord(e1, s);
      pending.push_back({kind, {e0, e1}});
    }
    ++count;
    return 0;
  }
  int go(const KInfo& k, long long work_lines, void** args, int kind = K_OP) {
    if (!k.fn || k.max_active <= 0) {
      g_err = "kernel configuration unavailable on this device (shared memory)";
      return 1;
    }
    long long need = (work_lines + k.lines - 1) / k.lines;
    long long cap = (long long)k.max_active * num_sms;
    unsigned grid = (unsigned)(need < cap ? need : cap);
    if (grid < 1) grid = 1;
    return raw(k.fn, grid, k.threads, k.smem, args, kind);
  }
};

template <class F>
int launch_elementwise(F* fn, Launcher& L, long long total, Args& a, int kind) {
  void* args[] = {&a};
  int per = 256;
  long long need = (total + per - 1) / per;
  long long cap = (long long)L.num_sms * 8;
  unsigned grid = (unsigned)(need < cap ? need : cap);
  if (grid < 1) grid = 1;
  return L.raw((const void*)fn, grid, per, 0, args, kind);
}

// Body-graph tail of the device-side WHILE loop: keep iterating until the
// monitor (solvers.py:243-277, run by the last CTA of the projection sweep)
// raises the stop flag.
__global__ void k_loop_cond(cudaGraphConditionalHandle h, const DevState* st) {
  cudaGraphSetConditional(h, st->stopped ? 0u : 1u);
}

// distributed solve: install global totals, then run the stopping monitor
__global__ void k_dist_monitor(Args a, const double* __restrict__ tot) {
  if (threadIdx.x || blockIdx.x) return;
  for (int c = 0; c < a.d; ++c) a.st->jmean[c] = make_double2(tot[2 * c], tot[2 * c + 1]);
  a.st->js2 = tot[6];
  monitor_step(a, tot[7] + tot[6]);
}
__global__ void k_dist_set_delta(Args a, const double* __restrict__ dl) {
  if (threadIdx.x || blockIdx.x) return;
  for (int c = 0; c < a.d; ++c) a.st->delta[c] = make_double2(dl[2 * c], dl[2 * c + 1]);
}

cudaStream_t capture_stream() {
  thread_local cudaStream_t cs = nullptr;
  if (!cs) cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  return cs;
}

}  // namespace

extern "C" {

const char* fftc_last_error(void) { return g_err.c_str(); }
int fftc_version(void) { return 100; }
int64_t fftc_launch_count(void) { return g_launches.load(); }
int32_t fftc_last_layout(void) { return g_last_zbs; }
int fftc_supported_length(int64_t n) { return even_axis(n) ? 1 : 0; }
int fftc_fused_length(int64_t n) { return lg2_exact(n) > 0 ? 1 : 0; }

void fftc_profile(int32_t enable) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_profile = enable != 0;
  for (auto& st : g_stats) st = KindStat();
}

int fftc_kernel_stats(fftc_kstat* out, int32_t max_entries) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  int n = 0;
  for (int k = 0; k < K_NKIND && n < max_entries; ++k) {
    if (!g_stats[k].launches) continue;
    snprintf(out[n].name, sizeof(out[n].name), "%s", kKindName[k]);
    out[n].launches = g_stats[k].launches;
    out[n].total_ms = g_stats[k].ms;
    ++n;
  }
  return n;
}

int fftc_solve(const fftc_problem* pb, const fftc_params* pr, double* history, int64_t history_cap,
               void* E, void* J, void* aug, fftc_result* out, void* stream) {
  g_err.clear();
  if (!pb || !pr || !out) {
    g_err = "null argument";
    return 2;
  }
  const int d = pb->d;
  if (d != 2 && d != 3) {
    g_err = "d must be 2 or 3";
    return 2;
  }
  const long long nx = pb->n[0], ny = pb->n[1], nz = d == 3 ? pb->n[2] : 1;
  if (!even_axis(nx) || !even_axis(ny) || (d == 3 && !even_axis(nz))) {
    g_err = "unsupported grid: every axis must be even and >= 2 (reference geometry.py:37)";
    return 3;
  }
  // powers of two 2..4096 run the fused sweeps; other even lengths (or
  // FFTC_GENERAL=1) the general path of general.cuh around cuFFT
  const bool general = general_grid(d, nx, ny, nz);
  const int lgx = general ? 1 : lg2_exact(nx), lgy = general ? 1 : lg2_exact(ny),
            lgz = general ? (d == 3 ? 1 : 0) : (d == 3 ? lg2_exact(nz) : 0);
  if (pr->scheme < 0 || pr->scheme > 3) {
    g_err = "bad scheme";
    return 2;
  }
  if (ensure_registry()) return 1;
  Registry& R = reg();
  cudaStream_t s = (cudaStream_t)stream;
  const long long N = nx * ny * nz;
  const int scheme = pr->scheme;
  const bool aug_s = scheme >= 2;

  // ---- scalars (host side, mirroring the reference expressions) ----
  Args a;
  memset(&a, 0, sizeof(a));
  a.d = d;
  a.nx = (int)nx;
  a.ny = (int)ny;
  a.nz = (int)nz;
  a.N = N;
  a.chi = pb->chi;
  a.row_e = row_e((int)nx, (int)scheme);
  fill_scalars(a, pr, d, N);

  // ---- workspace ----
  const int nslots = scheme == FFTC_EM_SUB ? 3 : (scheme == FFTC_BASIC_SUB ? 2 : 1);
  const size_t fld = sizeof(double2) * (size_t)d * N;
  bool use_graph;
  {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    // (FFTC_DEBUG_SYNC synchronises after every launch: not allowed in a capture)
    use_graph = !general && !g_profile && pr->max_iters <= (1 << 20) && !getenv("FFTC_NO_GRAPH") && !debug_sync();
  }
  // graph mode runs the whole loop in one launch: the device keeps every record
  const int hist_ring = use_graph ? (int)std::max<int64_t>(std::min<int64_t>(pr->max_iters, 1 << 20), 16) : 1024;
  const size_t partial_cap = (size_t)R.num_sms * 64 * NQMAX + 16 * NQMAX;
  char* ws = nullptr;
  char* ws_lean = nullptr;  // per-row compact offsets of the memory-lean schedule
  const bool two_work = (scheme == FFTC_EM || scheme == FFTC_EM_SUB);  // B holds the flux transform
  const bool chi_perm = !general && nx >= 16;  // thread-blocked chi rows for the TMA row sweeps
  const size_t small_bytes = sizeof(double) * partial_cap + sizeof(double) * 3 * hist_ring + sizeof(DevState) +
                             sizeof(int2) * (size_t)ny * nz + 8192;
  size_t ws_bytes = fld * (nslots + (two_work ? 2 : 1)) + small_bytes + (chi_perm ? (size_t)N + 256 : 0);
  // Memory-lean em_sub schedule (3-D, TMA row and column passes): S/T slots
  // compacted to the phase-1 voxels, and the flux transform Jq run on its own
  // ahead of the residual field's, through ONE work field: per voxel
  // 16d (Q) + 2*16d*f (S, T) + 16d (A) + 2 (rank codes) bytes instead of
  // 5*16d + 1 -- at 1024^3 with f = 0.3, 137 GB instead of 259 GB (SURVEY 7,
  // "memory at 1024^3").  Chosen when the normal workspace does not fit the
  // free device memory; FFTC_LEAN=1/0 forces it on/off.  Results are bit
  // identical to the normal schedule (same arithmetic, reordered launches).
  const LTable& TXl = R.tab[lgx];
  const bool lean_ok = scheme == FFTC_EM_SUB && d == 3 && !general && nx >= 512 && ny >= 256 && ny <= 1024 &&
                       nz >= 256 && nz <= 1024 && TXl.s1l[0].max_active > 0 && TXl.s1l[1].max_active > 0 &&
                       TXl.s3l.max_active > 0;
  bool lean = false;
  if (lean_ok) {
    if (const char* lv = getenv("FFTC_LEAN")) {
      lean = atoi(lv) != 0;
    } else {
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      if (ws_bytes + ((size_t)1 << 30) > fr) {  // cached pool blocks count as used: release them, ask again
        cudaMemPool_t pool;
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
          cudaStreamSynchronize(s);
          cudaMemPoolTrimTo(pool, 0);
        }
        cudaMemGetInfo(&fr, &tot);
        lean = ws_bytes + ((size_t)1 << 30) > fr;
      }
    }
  }
  long long M = 0;
  if (lean) {
    // phase-1 voxels per row -> exclusive offsets (host scan of ny*nz counts)
    const long long rows = ny * nz;
    CK(cudaMallocAsync((void**)&ws_lean, sizeof(long long) * (size_t)(rows + 1), s));
    {
      unsigned g = (unsigned)std::min<long long>((rows + 7) / 8, (long long)R.num_sms * 8);
      const uint8_t* chi = pb->chi;
      long long* cnt = (long long*)ws_lean;
      int nxi = (int)nx;
      void* ca[] = {(void*)&chi, (void*)&nxi, (void*)&rows, (void*)&cnt};
      CK(cudaLaunchKernel((const void*)k_row_counts, dim3(g), dim3(256), ca, 0, s));
    }
    std::vector<long long> off((size_t)rows + 1);
    CK(cudaMemcpyAsync(off.data(), ws_lean, sizeof(long long) * (size_t)rows, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    long long acc = 0;
    for (long long r = 0; r < rows; ++r) {
      const long long c = off[(size_t)r];
      off[(size_t)r] = acc;
      acc += c;
    }
    off[(size_t)rows] = acc;
    M = acc;
    CK(cudaMemcpyAsync(ws_lean, off.data(), sizeof(long long) * (size_t)(rows + 1), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));  // `off` leaves scope
    ws_bytes = 2 * fld + 2 * sizeof(double2) * (size_t)d * (size_t)std::max<long long>(M, 1) + small_bytes +
               2 * (size_t)N + 512;
  }
  CK(cudaMallocAsync((void**)&ws, ws_bytes, s));
  size_t o = 0;
  auto carve = [&](size_t bytes) {
    char* p = ws + o;
    o += (bytes + 255) & ~(size_t)255;
    return p;
  };
  if (lean) {
    const size_t cfld = sizeof(double2) * (size_t)d * (size_t)std::max<long long>(M, 1);
    a.X[0] = (double2*)carve(fld);
    a.X[1] = (double2*)carve(cfld);
    a.X[2] = (double2*)carve(cfld);
    a.A = a.B = (double2*)carve(fld);
    a.rowoff = (const long long*)ws_lean;
    a.M = M;
    a.chiR = (const uint16_t*)carve(2 * (size_t)N);
  } else {
    for (int i = 0; i < nslots; ++i) a.X[i] = (double2*)carve(fld);
    a.A = (double2*)carve(fld);
    a.B = two_work ? (double2*)carve(fld) : a.A;
  }
  a.partials = (double*)carve(sizeof(double) * partial_cap);
  a.history = (double*)carve(sizeof(double) * 3 * hist_ring);
  a.hist_cap = hist_ring;
  a.st = (DevState*)carve(sizeof(DevState));
  a.row_ext = (const int2*)carve(sizeof(int2) * (size_t)ny * nz);
  a.chiT = (chi_perm && !lean) ? (const uint8_t*)carve((size_t)N) : nullptr;
  a.dbg = getenv("FFTC_PHASE") ? (unsigned long long*)carve(sizeof(unsigned long long) * 8) : nullptr;
  if (a.dbg) CK(cudaMemsetAsync(a.dbg, 0, sizeof(unsigned long long) * 8, s));
  a.outE = (double2*)E;
  a.outJ = (double2*)J;
  a.outAug = (double2*)aug;
  a.tw[0] = R.tw[lgx];
  a.tw[1] = R.tw[lgy];
  a.tw[2] = d == 3 ? R.tw[lgz] : R.tw[lgy];

  int rc = 0;
  cudaEvent_t ev0, ev1;
  CK(cudaEventCreate(&ev0));
  CK(cudaEventCreate(&ev1));
  thread_local DevState* hst = nullptr;
  if (!hst) CK(cudaMallocHost((void**)&hst, sizeof(DevState)));
  Launcher Lc(s, R.num_sms);
  const LTable& TX = R.tab[lgx];
  const LTable& TY = R.tab[lgy];
  const LTable& TZ = R.tab[d == 3 ? lgz : lgy];
  long long nrec_host = 0;
  bool stopped = false;
  cufftHandle plan = 0;  // general path: batched d-component transform (cuFFT)

  do {
    if (general) {
      long long n[3];
      if (d == 2) {
        n[0] = ny;
        n[1] = nx;
      } else {
        n[0] = nz;
        n[1] = ny;
        n[2] = nx;
      }
      size_t wsz = 0;
      if (cufftCreate(&plan) != CUFFT_SUCCESS ||
          cufftMakePlanMany64(plan, d, n, nullptr, 1, N, nullptr, 1, N, CUFFT_Z2Z, d, &wsz) != CUFFT_SUCCESS) {
        g_err = "cuFFT plan for the general grid failed";
        rc = 1;
        break;
      }
    }
    CK(cudaMemsetAsync(a.st, 0, sizeof(DevState), s));
    CK(cudaEventRecord(ev0, s));
    {
      const long long rows = ny * nz;
      unsigned g = (unsigned)std::min<long long>((rows + 7) / 8, (long long)R.num_sms * 8);
      void* ea[] = {(void*)&a.chi, (void*)&a.nx, (void*)&rows, (void*)&a.row_ext};
      if ((rc = Lc.raw((const void*)k_row_extent, g, 256, 0, ea, K_INIT))) break;
      if (lean) {  // rank codes of the compact S/T slots
        void* ra[] = {(void*)&a.chi, (void*)&a.nx, (void*)&rows, (void*)&a.chiR, (void*)&a.row_e};
        if ((rc = Lc.raw((const void*)k_chi_rank16, g, 256, 0, ra, K_INIT))) break;
      } else if (chi_perm) {
        const long long chunks = rows * (nx / a.row_e);
        unsigned gp = (unsigned)std::min<long long>((chunks + 255) / 256, (long long)R.num_sms * 16);
        void* pa[] = {(void*)&a.chi, (void*)&a.nx, (void*)&rows, (void*)&a.chiT, (void*)&a.row_e};
        if ((rc = Lc.raw((const void*)k_chi_perm16, gp, 256, 0, pa, K_INIT))) break;
      }
    }
    switch (scheme) {
      case FFTC_BASIC: rc = launch_elementwise(k_init<BASIC>, Lc, (long long)d * N, a, K_INIT); break;
      case FFTC_EM: rc = launch_elementwise(k_init<EM>, Lc, (long long)d * N, a, K_INIT); break;
      case FFTC_BASIC_SUB: rc = launch_elementwise(k_init<BASIC_SUB>, Lc, (long long)d * N, a, K_INIT); break;
      default: rc = launch_elementwise(k_init<EM_SUB>, Lc, (long long)d * N, a, K_INIT); break;
    }
    if (rc) break;

    // column geometries
    ColGeom mid{};
    ColGeom yf{};
    CUtensorMap tmA, tmB;
    bool use_tma_mid = false;
    const bool em_type = (scheme == FFTC_EM || scheme == FFTC_EM_SUB);
    const KInfo* kmid;
    if (d == 2) {
      mid.axis = 1;
      mid.nouter = 1;
      mid.stride = nx;
      mid.ostride = 0;
      mid.nstrips = (int)(nx / TY.col_w);
      kmid = &TY.col[em_type ? KC_MID2_EM : KC_MID2_BASIC];
      const KInfo& kt = TY.col[em_type ? KC_MID2T_EM : KC_MID2T_BASIC];
      if (kt.fn && kt.max_active > 0 && !getenv("FFTC_NO_TMA_COLS") &&
          make_field_map(&tmA, a.A, nx, ny, d, ny < 256 ? (int)ny : 256) &&
          make_field_map(&tmB, a.B, nx, ny, d, ny < 256 ? (int)ny : 256)) {
        kmid = &kt;
        use_tma_mid = true;
      }
    } else {
      mid.axis = 2;
      mid.nouter = (int)ny;
      mid.stride = nx * ny;
      mid.ostride = nx;
      mid.nstrips = (int)(nx / TZ.col3_w);
      mid.o0 = 0;
      mid.on = (int)ny;
      kmid = &TZ.col[em_type ? KC_MID3_EM : KC_MID3_BASIC];
      yf.axis = 1;
      yf.nouter = (int)nz;
      yf.stride = nx;
      yf.ostride = nx * ny;
      yf.nstrips = (int)(nx / 2);
    }
    // 3-D TMA column passes (cols3_lg.cuh) where the line lengths allow
    Col3Pass zmid, yfwd, yinv, zpar;
    const PeerOut* no_peer = nullptr;
    a.zbs = 0;
    g_last_zbs = 0;
    if (lean) {
      // one work field: y forward and the projection pass on A alone; the
      // residual pass reads A through the "flux field" map (every tile
      // Parseval-only, f0 = 1) and runs the monitor; the residual field's
      // projection pass leaves the monitor alone
      const int zbs = zblock_shift(nx, ny, nz);
      const KInfo& kz = TZ.col[KC_MID3T_EM];
      if (!(zbs > 0 && col3_pass_zblk(zpar, kz, a, a.A, a.A, 2, zbs, 1) &&
            col3_pass_zblk(zmid, kz, a, a.A, nullptr, 2, zbs, 1) &&
            col3_pass_zblk(yfwd, TY.col[KC_FWD3T], a, a.A, nullptr, 1, zbs, 1) &&
            col3_pass_zblk(yinv, TY.col[KC_INV3T], a, a.A, nullptr, 1, zbs, 1))) {
        g_err = "memory-lean em_sub schedule: the z-blocked TMA column passes are unavailable for this grid";
        rc = 3;
        break;
      }
      zpar.g.f0 = 1;
      zmid.g.no_monitor = 1;
      a.zbs = zbs;
      g_last_zbs = zbs | 256;
    } else if (d == 3 && !general) {
      // z-blocked work fields when all three column passes run on TMA tiles
      const int zbs = zblock_shift(nx, ny, nz);
      const KInfo& kz = TZ.col[em_type ? KC_MID3T_EM : KC_MID3T_BASIC];
      if (zbs > 0 && col3_pass_zblk(zmid, kz, a, a.A, em_type ? a.B : nullptr, 2, zbs, em_type ? 2 : 1) &&
          col3_pass_zblk(yfwd, TY.col[KC_FWD3T], a, a.A, em_type ? a.B : nullptr, 1, zbs, em_type ? 2 : 1) &&
          col3_pass_zblk(yinv, TY.col[KC_INV3T], a, a.A, nullptr, 1, zbs, 1)) {
        a.zbs = zbs;
        g_last_zbs = zbs;
      } else {
        col3_pass(zmid, kz, a, a.A, em_type ? a.B : nullptr, nz, nx * ny, ny, nx, N, em_type ? 2 : 1, 2, 0, (int)ny);
        col3_pass(yfwd, TY.col[KC_FWD3T], a, a.A, em_type ? a.B : nullptr, ny, nx, nz, nx * ny, N, em_type ? 2 : 1, 1,
                  0, (int)nz);
        col3_pass(yinv, TY.col[KC_INV3T], a, a.A, nullptr, ny, nx, nz, nx * ny, N, 1, 1, 0, (int)nz);
      }
    }
    const long long mid_lines = use_tma_mid ? nx * (em_type ? 2 : 1)
                                            : (long long)mid.nouter * mid.nstrips * (em_type ? 2 : 1);
    const long long row_lines = (long long)d * ny * nz;
    const long long yf_lines = (long long)yf.nouter * yf.nstrips * d;
    void* a1[] = {&a};
    void* amid_std[] = {&a, &mid};
    void* amid_tma[] = {&a, &tmA, &tmB};
    void** amid = use_tma_mid ? amid_tma : amid_std;
    ColGeom yfB = yf;  // forward y pass of field B (em-type) uses the same geometry

    // general grids: prologue, cuFFT forward, Gamma^ + monitor, cuFFT
    // inverse, epilogue (general.cuh)
    auto launch_gen = [&](Launcher& L) -> int {
      int r = 0;
      switch (scheme) {
        case FFTC_BASIC: r = launch_elementwise(k_gen_pro<BASIC>, L, (long long)d * N, a, K_SWEEP1); break;
        case FFTC_EM: r = launch_elementwise(k_gen_pro<EM>, L, (long long)d * N, a, K_SWEEP1); break;
        case FFTC_BASIC_SUB: r = launch_elementwise(k_gen_pro<BASIC_SUB>, L, (long long)d * N, a, K_SWEEP1); break;
        default: r = launch_elementwise(k_gen_pro<EM_SUB>, L, (long long)d * N, a, K_SWEEP1); break;
      }
      if (r) return r;
      if (cufftSetStream(plan, L.s) != CUFFT_SUCCESS ||
          cufftExecZ2Z(plan, (cufftDoubleComplex*)a.A, (cufftDoubleComplex*)a.A, CUFFT_FORWARD) != CUFFT_SUCCESS ||
          (em_type &&
           cufftExecZ2Z(plan, (cufftDoubleComplex*)a.B, (cufftDoubleComplex*)a.B, CUFFT_FORWARD) != CUFFT_SUCCESS)) {
        g_err = "cuFFT forward transform failed";
        return 1;
      }
      r = em_type ? launch_elementwise(k_gen_gamma<MID_EM>, L, N, a, K_MID)
                  : launch_elementwise(k_gen_gamma<MID_BASIC>, L, N, a, K_MID);
      if (r) return r;
      if (cufftExecZ2Z(plan, (cufftDoubleComplex*)a.A, (cufftDoubleComplex*)a.A, CUFFT_INVERSE) != CUFFT_SUCCESS) {
        g_err = "cuFFT inverse transform failed";
        return 1;
      }
      switch (scheme) {
        case FFTC_BASIC: return launch_elementwise(k_gen_epi<BASIC>, L, (long long)d * N, a, K_SWEEP3);
        case FFTC_EM: return launch_elementwise(k_gen_epi<EM>, L, (long long)d * N, a, K_SWEEP3);
        case FFTC_BASIC_SUB: return launch_elementwise(k_gen_epi<BASIC_SUB>, L, (long long)d * N, a, K_SWEEP3);
        default: return launch_elementwise(k_gen_epi<EM_SUB>, L, (long long)d * N, a, K_SWEEP3);
      }
    };

    // memory-lean em_sub iteration (solvers.py:395-432 in two halves): the
    // flux Jq's forward transform and residual (Parseval) with the monitor,
    // then -- unless stopped -- the residual field Rq's transform, (I - 2
    // Gamma^), inverse and the state update, all through work field A
    auto launch_lean = [&](Launcher& L) -> int {
      int r;
      void* ay[] = {&a, &yfwd.g, &yfwd.mA, &yfwd.mB, &no_peer};
      void* azp[] = {&a, &zpar.g, &zpar.mA, &zpar.mB, &no_peer};
      void* azm[] = {&a, &zmid.g, &zmid.mA, &zmid.mB, &no_peer};
      void* ayi[] = {&a, &yinv.g, &yinv.mA, &yinv.mB, &no_peer};
      if ((r = L.go(TX.s1l[0], row_lines, a1, K_SWEEP1))) return r;
      if ((r = L.go(*yfwd.k, yfwd.tiles, ay, K_YFWD))) return r;
      if ((r = L.go(*zpar.k, zpar.tiles, azp, K_PARSEVAL))) return r;
      if ((r = L.go(TX.s1l[1], row_lines, a1, K_SWEEP1))) return r;
      if ((r = L.go(*yfwd.k, yfwd.tiles, ay, K_YFWD))) return r;
      if ((r = L.go(*zmid.k, zmid.tiles, azm, K_MID))) return r;
      if ((r = L.go(*yinv.k, yinv.tiles, ayi, K_YINV))) return r;
      return L.go(TX.s3l, row_lines, a1, K_SWEEP3);
    };

    // one reference iteration (solvers.py:300-321 / :395-432) = these launches
    auto launch_iter = [&](Launcher& L) -> int {
      if (general) return launch_gen(L);
      if (lean) return launch_lean(L);
      int r = L.go(TX.s1[scheme], row_lines, a1, K_SWEEP1);
      if (r) return r;
      if (d == 3) {
        // y forward of field A (and B for em-type)
        if (yfwd.ok) {
          void* ay[] = {&a, &yfwd.g, &yfwd.mA, &yfwd.mB, &no_peer};
          if ((r = L.go(*yfwd.k, yfwd.tiles, ay, K_YFWD))) return r;
          // timing experiments only (results wrong): the pass once more right after
          // itself (1), or the inverse-pass kernel on the same tiles (2)
          if (const char* e = getenv("FFTC_DBG_YFWD2")) {
            const KInfo& kk = atoi(e) == 2 ? TY.col[KC_INV3T] : *yfwd.k;
            if ((r = L.go(kk, yfwd.tiles, ay, K_PARSEVAL))) return r;
          }
        } else {
          Args aB = a;
          void* ayf[] = {&a, &yf};
          if ((r = L.go(TY.col[KC_FWD], yf_lines, ayf, K_YFWD))) return r;
          if (em_type) {
            aB.A = a.B;
            void* ab[] = {&aB, &yfB};
            if ((r = L.go(TY.col[KC_FWD], yf_lines, ab, K_YFWD))) return r;
          }
        }
      }
      if (d == 3 && zmid.ok) {
        void* az[] = {&a, &zmid.g, &zmid.mA, &zmid.mB, &no_peer};
        if ((r = L.go(*zmid.k, zmid.tiles, az, K_MID))) return r;
      } else if ((r = L.go(*kmid, mid_lines, amid, K_MID))) {
        return r;
      }
      if (d == 3) {
        if (yinv.ok) {
          void* ay[] = {&a, &yinv.g, &yinv.mA, &yinv.mB, &no_peer};
          if ((r = L.go(*yinv.k, yinv.tiles, ay, K_YINV))) return r;
        } else {
          void* ai[] = {&a, &yf};
          if ((r = L.go(TY.col[KC_INV], yf_lines, ai, K_YINV))) return r;
        }
      }
      return L.go(TX.s3[scheme], row_lines, a1, K_SWEEP3);
    };

    if (use_graph) {
      // CUDA graph with a conditional WHILE node: the body is one iteration
      // plus k_loop_cond; the whole solve is a single graph launch and the
      // host never synchronises inside the loop.
      cudaGraph_t g = nullptr, body = nullptr;
      cudaGraphExec_t ge = nullptr;
      cudaGraphConditionalHandle h;
      cudaStream_t cs = capture_stream();
      long long per_iter_launches = 0;
      do {
        if ((rc = (cudaGraphCreate(&g, 0) != cudaSuccess))) break;
        if ((rc = (cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault) != cudaSuccess))) break;
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t cn;
        if ((rc = (cudaGraphAddNode(&cn, g, nullptr, 0, &cp) != cudaSuccess))) break;
        body = cp.conditional.phGraph_out[0];
        if ((rc = (cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed) !=
                   cudaSuccess)))
          break;
        Launcher Lcap(cs, R.num_sms);
        int r1 = launch_iter(Lcap);
        per_iter_launches = Lcap.count + 1;  // + the condition kernel below
        const DevState* stp = a.st;
        void* ca[] = {&h, &stp};
        if (!r1) r1 = Lcap.raw((const void*)k_loop_cond, 1, 1, 0, ca, K_OP);
        cudaGraph_t cap_out = nullptr;
        cudaError_t ec = cudaStreamEndCapture(cs, &cap_out);
        Lc.count += 0;
        if (r1 || ec != cudaSuccess) {
          rc = r1 ? r1 : 1;
          break;
        }
        if ((rc = (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess))) break;
        if ((rc = (cudaGraphLaunch(ge, s) != cudaSuccess))) break;
      } while (0);
      if (rc && g_err.empty()) g_err = std::string("graph loop: ") + cudaGetErrorString(cudaGetLastError());
      if (!rc) {
        CK(cudaMemcpyAsync(hst, a.st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const long long nrec = hst->nrec;
        if (nrec > history_cap) {
          g_err = "history buffer too small";
          rc = 4;
        } else if (nrec > 0) {
          CK(cudaMemcpy(history, a.history, sizeof(double) * 3 * nrec, cudaMemcpyDeviceToHost));
        }
        // launches executed by the loop: (kernels per body) x iterations run
        Lc.count += per_iter_launches * std::max<long long>(hst->k, 1);
      }
      if (ge) cudaGraphExecDestroy(ge);
      if (g) cudaGraphDestroy(g);
      if (rc) break;
    } else {
      // profiling: one iteration per synchronisation, so no launch after the
      // stop is counted in the per-kernel statistics
      long long chunk = Lc.prof ? 1 : 2;
      const long long max_chunk = Lc.prof ? 1 : 256;
      long long launched_iters = 0;
      while (!stopped) {
        long long todo = chunk;
        if (launched_iters + todo > pr->max_iters) todo = pr->max_iters - launched_iters;
        for (long long it = 0; it < todo && !rc; ++it) rc = launch_iter(Lc);
        if (rc) break;
        launched_iters += todo;
        CK(cudaMemcpyAsync(hst, a.st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        Lc.harvest();
        // collect new history records from the device ring
        long long nrec = hst->nrec;
        if (nrec > history_cap) {
          g_err = "history buffer too small";
          rc = 4;
          break;
        }
        for (long long r0 = nrec_host; r0 < nrec;) {
          long long slot = r0 % hist_ring;
          long long cnt = std::min(nrec - r0, (long long)hist_ring - slot);
          CK(cudaMemcpy(history + 3 * r0, a.history + 3 * slot, sizeof(double) * 3 * cnt, cudaMemcpyDeviceToHost));
          r0 += cnt;
        }
        nrec_host = nrec;
        stopped = hst->stopped != 0 || launched_iters >= pr->max_iters;
        chunk = std::min<long long>(chunk * 2, max_chunk);
      }
    }
    if (rc) break;
    switch (scheme) {
      case FFTC_BASIC: rc = launch_elementwise(k_finalize<BASIC>, Lc, (long long)d * N, a, K_FINAL); break;
      case FFTC_EM: rc = launch_elementwise(k_finalize<EM>, Lc, (long long)d * N, a, K_FINAL); break;
      case FFTC_BASIC_SUB: rc = launch_elementwise(k_finalize<BASIC_SUB>, Lc, (long long)d * N, a, K_FINAL); break;
      default: rc = launch_elementwise(k_finalize<EM_SUB>, Lc, (long long)d * N, a, K_FINAL); break;
    }
    if (rc) break;
    CK(cudaEventRecord(ev1, s));
    CK(cudaMemcpyAsync(hst, a.st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ev0, ev1));
    if (a.dbg) {
      unsigned long long hd[8];
      CK(cudaMemcpy(hd, a.dbg, sizeof(hd), cudaMemcpyDeviceToHost));
      unsigned long long tot = 0;
      for (int i = 0; i < 8; ++i) tot += hd[i];
      fprintf(stderr, "[fftc phase cycles] loop %.1f%% tma-wait %.1f%% lds-in %.1f%% fwd %.1f%% proj %.1f%% inv %.1f%% store %.1f%% issue %.1f%%\n",
              100.0 * hd[0] / tot, 100.0 * hd[1] / tot, 100.0 * hd[2] / tot, 100.0 * hd[3] / tot, 100.0 * hd[4] / tot,
              100.0 * hd[5] / tot, 100.0 * hd[6] / tot, 100.0 * hd[7] / tot);
    }
    out->device_ms = ms;
    out->status = hst->status;
    out->degenerate_flux = hst->degenerate;
    out->iterations = hst->nrec;
    if (hst->nrec > 0) {
      out->sigma_star[0] = history[3 * (hst->nrec - 1) + 0];
      out->sigma_star[1] = history[3 * (hst->nrec - 1) + 1];
    } else {
      out->sigma_star[0] = hst->last_sstar.x;
      out->sigma_star[1] = hst->last_sstar.y;
    }
    for (int c = 0; c < 3; ++c) {
      out->mean_E[c][0] = c < d ? hst->meanE[c].x : 0.0;
      out->mean_E[c][1] = c < d ? hst->meanE[c].y : 0.0;
      out->mean_J[c][0] = c < d ? hst->meanJ[c].x : 0.0;
      out->mean_J[c][1] = c < d ? hst->meanJ[c].y : 0.0;
    }
  } while (0);
  if (plan) {
    cudaStreamSynchronize(s);  // the plan's work area may still be in use
    cufftDestroy(plan);
  }
  out->kernel_launches = Lc.count;
  g_launches += Lc.count;
  cudaFreeAsync(ws, s);
  if (ws_lean) cudaFreeAsync(ws_lean, s);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  if (!rc) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      g_err = cudaGetErrorString(e);
      rc = 1;
    }
  }
  return rc;
}

// ---------------------------------------------------------------------------
// operator API: plain transforms and the Gamma_1 projection on device fields
// ---------------------------------------------------------------------------
namespace {
struct GridInfo {
  int d, lgx, lgy, lgz;
  long long nx, ny, nz, N;
  bool general;  // an axis outside the fused lengths: cuFFT + general.cuh
};
int grid_info(const fftc_problem* pb, GridInfo& g) {
  if (!pb || (pb->d != 2 && pb->d != 3)) {
    g_err = "d must be 2 or 3";
    return 2;
  }
  g.d = pb->d;
  g.nx = pb->n[0];
  g.ny = pb->n[1];
  g.nz = g.d == 3 ? pb->n[2] : 1;
  if (!even_axis(g.nx) || !even_axis(g.ny) || (g.d == 3 && !even_axis(g.nz))) {
    g_err = "unsupported grid: every axis must be even and >= 2 (reference geometry.py:37)";
    return 3;
  }
  g.general = general_grid(g.d, g.nx, g.ny, g.nz);
  g.lgx = g.general ? 1 : lg2_exact(g.nx);
  g.lgy = g.general ? 1 : lg2_exact(g.ny);
  g.lgz = g.d == 3 ? (g.general ? 1 : lg2_exact(g.nz)) : 0;
  g.N = g.nx * g.ny * g.nz;
  return 0;
}

// general grids: unnormalised cuFFT transforms of a (d, grid) field in place,
// all axes (mask 2^d - 1: one batched rank-d plan) or axis by axis
int cufft_axes(double2* data, const GridInfo& g, int mask, bool inverse, cudaStream_t s) {
  const int dir = inverse ? CUFFT_INVERSE : CUFFT_FORWARD;
  auto run = [&](int rank, long long* n, long long istride, long long idist, long long batch, long long nblocks,
                 long long bstride) -> int {
    cufftHandle plan = 0;
    size_t wsz = 0;
    int rc = 0;
    if (cufftCreate(&plan) != CUFFT_SUCCESS ||
        cufftMakePlanMany64(plan, rank, n, n, istride, idist, n, istride, idist, CUFFT_Z2Z, batch, &wsz) !=
            CUFFT_SUCCESS ||
        cufftSetStream(plan, s) != CUFFT_SUCCESS) {
      g_err = "cuFFT plan failed";
      rc = 1;
    }
    for (long long b = 0; !rc && b < nblocks; ++b) {
      cufftDoubleComplex* p = (cufftDoubleComplex*)(data + b * bstride);
      if (cufftExecZ2Z(plan, p, p, dir) != CUFFT_SUCCESS) {
        g_err = "cuFFT transform failed";
        rc = 1;
      }
    }
    if (plan) {
      cudaStreamSynchronize(s);  // the plan's work area may still be in use
      cufftDestroy(plan);
    }
    return rc;
  };
  const int all = (1 << g.d) - 1;
  if ((mask & all) == all) {
    long long n[3];
    if (g.d == 2) {
      n[0] = g.ny;
      n[1] = g.nx;
    } else {
      n[0] = g.nz;
      n[1] = g.ny;
      n[2] = g.nx;
    }
    return run(g.d, n, 1, g.N, g.d, 1, 0);
  }
  for (int ax = 0; ax < g.d; ++ax) {
    if (!(mask & (1 << ax))) continue;
    long long n[1] = {ax == 0 ? g.nx : (ax == 1 ? g.ny : g.nz)};
    const long long stride = ax == 0 ? 1 : (ax == 1 ? g.nx : g.nx * g.ny);
    const long long block = n[0] * stride;  // contiguous elements holding `stride` interleaved lines
    const long long nblocks = (long long)g.d * g.N / block;
    int rc = stride == 1 ? run(1, n, 1, n[0], nblocks, 1, 0) : run(1, n, stride, 1, stride, nblocks, block);
    if (rc) return rc;
  }
  return 0;
}

// scratch state for kernels that end in a reduction
struct Scratch {
  char* ws = nullptr;
  cudaStream_t s = nullptr;
  int alloc(Args& a, int num_sms, cudaStream_t st) {
    s = st;
    const size_t pc = (size_t)num_sms * 64 * NQMAX + 16 * NQMAX;
    const size_t bytes = sizeof(double) * pc + sizeof(double) * 3 * 16 + sizeof(DevState) + 1024;
    CK(cudaMallocAsync((void**)&ws, bytes, s));
    CK(cudaMemsetAsync(ws, 0, bytes, s));
    a.partials = (double*)ws;
    a.history = (double*)(ws + ((sizeof(double) * pc + 255) & ~(size_t)255));
    a.hist_cap = 16;
    a.st = (DevState*)((char*)a.history + 512);
    return 0;
  }
  ~Scratch() {
    if (ws) cudaFreeAsync(ws, s);
  }
};

int run_axis(Launcher& Lc, Args& a, const GridInfo& g, int axis, bool inverse, double scale) {
  Registry& R = reg();
  if (axis == 0) {
    const KInfo& k = inverse ? R.tab[g.lgx].row_inv : R.tab[g.lgx].row_fwd;
    void* args[] = {&a, &scale};
    return Lc.go(k, (long long)g.d * g.ny * g.nz, args);
  }
  ColGeom gm{};
  int lg;
  if (axis == 1) {
    lg = g.lgy;
    gm.axis = 1;
    gm.nouter = (int)g.nz;
    gm.stride = g.nx;
    gm.ostride = g.nx * g.ny;
  } else {
    lg = g.lgz;
    gm.axis = 2;
    gm.nouter = (int)g.ny;
    gm.stride = g.nx * g.ny;
    gm.ostride = g.nx;
  }
  gm.nstrips = (int)(g.nx / 2);
  void* args[] = {&a, &gm};
  const KInfo& k = R.tab[lg].col[inverse ? KC_INV : KC_FWD];
  return Lc.go(k, (long long)gm.nouter * gm.nstrips * g.d, args);
}
}  // namespace

int fftc_fft(const fftc_problem* pb, void* data, int32_t inverse, int32_t axes_mask, void* stream) {
  g_err.clear();
  GridInfo g;
  if (int rc = grid_info(pb, g)) return rc;
  if (ensure_registry()) return 1;
  Registry& R = reg();
  Args a;
  memset(&a, 0, sizeof(a));
  a.d = g.d;
  a.nx = (int)g.nx;
  a.ny = (int)g.ny;
  a.nz = (int)g.nz;
  a.N = g.N;
  a.A = (double2*)data;
  a.op_mode = 1;
  a.tw[0] = R.tw[g.lgx];
  a.tw[1] = R.tw[g.lgy];
  a.tw[2] = g.d == 3 ? R.tw[g.lgz] : R.tw[g.lgy];
  cudaStream_t s = (cudaStream_t)stream;
  if (g.general) {
    if (int rc = cufft_axes((double2*)data, g, axes_mask, inverse != 0, s)) return rc;
    CK(cudaGetLastError());
    return 0;
  }
  Scratch sc;
  if (sc.alloc(a, R.num_sms, s)) return 1;
  Launcher Lc(s, R.num_sms);
  for (int ax = 0; ax < g.d; ++ax)
    if (axes_mask & (1 << ax))
      if (int rc = run_axis(Lc, a, g, ax, inverse != 0, 1.0)) return rc;
  g_launches += Lc.count;
  CK(cudaGetLastError());
  return 0;
}

int fftc_gamma1(const fftc_problem* pb, const void* in, void* out, double scale, void* stream) {
  g_err.clear();
  GridInfo g;
  if (int rc = grid_info(pb, g)) return rc;
  if (ensure_registry()) return 1;
  Registry& R = reg();
  cudaStream_t s = (cudaStream_t)stream;
  Args a;
  memset(&a, 0, sizeof(a));
  a.d = g.d;
  a.nx = (int)g.nx;
  a.ny = (int)g.ny;
  a.nz = (int)g.nz;
  a.N = g.N;
  a.inv_n = 1.0 / (double)g.N;
  a.gscale = scale;
  a.A = (double2*)out;
  a.B = (double2*)out;
  a.tw[0] = R.tw[g.lgx];
  a.tw[1] = R.tw[g.lgy];
  a.tw[2] = g.d == 3 ? R.tw[g.lgz] : R.tw[g.lgy];
  a.op_mode = 1;
  if (in != out) CK(cudaMemcpyAsync(out, in, sizeof(double2) * g.d * g.N, cudaMemcpyDeviceToDevice, s));
  Scratch sc;
  if (sc.alloc(a, R.num_sms, s)) return 1;
  Launcher Lc(s, R.num_sms);
  if (g.general) {  // cuFFT forward, Gamma^ (scaled by 1/N in operator mode), cuFFT inverse
    const int all = (1 << g.d) - 1;
    int rc = cufft_axes(a.A, g, all, false, s);
    if (!rc) rc = launch_elementwise(k_gen_gamma<MID_BASIC>, Lc, g.N, a, K_OP);
    if (!rc) rc = cufft_axes(a.A, g, all, true, s);
    g_launches += Lc.count;
    if (rc) return rc;
    CK(cudaGetLastError());
    return 0;
  }
  int rc = run_axis(Lc, a, g, 0, false, 1.0);
  if (!rc && g.d == 3) rc = run_axis(Lc, a, g, 1, false, 1.0);
  if (!rc) {
    ColGeom mid{};
    const KInfo* kmid;
    if (g.d == 2) {
      mid.axis = 1;
      mid.nouter = 1;
      mid.stride = g.nx;
      mid.nstrips = (int)(g.nx / R.tab[g.lgy].col_w);
      kmid = &R.tab[g.lgy].col[KC_MID2_BASIC];
    } else {
      mid.axis = 2;
      mid.nouter = (int)g.ny;
      mid.stride = g.nx * g.ny;
      mid.ostride = g.nx;
      mid.nstrips = (int)(g.nx / R.tab[g.lgz].col3_w);
      mid.o0 = 0;
      mid.on = (int)g.ny;
      kmid = &R.tab[g.lgz].col[KC_MID3_BASIC];
    }
    void* args[] = {&a, &mid};
    rc = Lc.go(*kmid, (long long)mid.nouter * mid.nstrips, args);
  }
  if (!rc && g.d == 3) rc = run_axis(Lc, a, g, 1, true, 1.0);
  if (!rc) rc = run_axis(Lc, a, g, 0, true, a.inv_n);
  g_launches += Lc.count;
  if (rc) return rc;
  CK(cudaGetLastError());
  return 0;
}

// test hook: run only the projection sweep (line FFT, Gamma, inverse line
// FFT along y in 2-D / z in 3-D) on a field already transformed along the
// other axes.
int fftc_debug_project(const fftc_problem* pb, void* data, void* stream) {
  g_err.clear();
  GridInfo g;
  if (int rc = grid_info(pb, g)) return rc;
  if (g.general) {
    g_err = "fftc_debug_project: fused (power-of-two) lengths only";
    return 3;
  }
  if (ensure_registry()) return 1;
  Registry& R = reg();
  cudaStream_t s = (cudaStream_t)stream;
  Args a;
  memset(&a, 0, sizeof(a));
  a.d = g.d;
  a.nx = (int)g.nx;
  a.ny = (int)g.ny;
  a.nz = (int)g.nz;
  a.N = g.N;
  a.inv_n = 1.0 / (double)g.N;
  a.gscale = 1.0;
  a.A = a.B = (double2*)data;
  a.op_mode = 1;
  a.tw[0] = R.tw[g.lgx];
  a.tw[1] = R.tw[g.lgy];
  a.tw[2] = g.d == 3 ? R.tw[g.lgz] : R.tw[g.lgy];
  Scratch sc;
  if (sc.alloc(a, R.num_sms, s)) return 1;
  Launcher Lc(s, R.num_sms);
  ColGeom mid{};
  const KInfo* kmid;
  if (g.d == 2) {
    mid.axis = 1;
    mid.nouter = 1;
    mid.stride = g.nx;
    mid.nstrips = (int)(g.nx / R.tab[g.lgy].col_w);
    kmid = &R.tab[g.lgy].col[KC_MID2_BASIC];
  } else {
    mid.axis = 2;
    mid.nouter = (int)g.ny;
    mid.stride = g.nx * g.ny;
    mid.ostride = g.nx;
    mid.nstrips = (int)(g.nx / R.tab[g.lgz].col3_w);
    mid.o0 = 0;
    mid.on = (int)g.ny;
    kmid = &R.tab[g.lgz].col[KC_MID3_BASIC];
  }
  void* args[] = {&a, &mid};
  if (int rc = Lc.go(*kmid, (long long)mid.nouter * mid.nstrips, args)) return rc;
  CK(cudaStreamSynchronize(s));
  return 0;
}

// Batched sweep (BASELINE config 5): n_points independent solves on one
// grid, run back to back on one stream (the workspace comes from the warm
// stream-ordered pool, so per-point setup is a few microseconds).
int fftc_solve_batch(const fftc_problem* pb, const fftc_params* params, int32_t n_points, double* histories,
                     int64_t history_cap, fftc_result* out, void* stream) {
  g_err.clear();
  if (!params || !out || n_points < 0) {
    g_err = "null argument";
    return 2;
  }
  // Points are independent solves.  Small and medium grids leave the GPU
  // idle between a solve's kernels (launch tails, the per-solve setup and
  // read-back), so several points run concurrently, one host worker and one
  // non-blocking stream each (FFTC_BATCH_STREAMS, default 8; 1 = in order;
  // C5 at 1024^2: 4 -> 9.36, 8 -> 9.66 G vox-it/s).
  // Every solve is deterministic on its own, so the results do not depend on
  // the interleaving.
  int width = 8;
  if (const char* e = getenv("FFTC_BATCH_STREAMS")) width = std::max(1, atoi(e));
  width = std::min<int>(width, std::max<int32_t>(n_points, 1));
  {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (g_profile) width = 1;  // per-kernel statistics are collected in launch order
  }
  if (width > 1 && pb) {
    // every concurrent point holds its own workspace (state slots + work
    // fields, fftc_solve): run only as many at once as the free device
    // memory holds, down to one at a time for large grids (a 512^3 em_sub
    // point alone needs ~32 GB)
    const long long N = pb->n[0] * pb->n[1] * (pb->d == 3 ? pb->n[2] : 1);
    size_t per = 0;
    for (int32_t i = 0; i < n_points; ++i) {
      const int sc = params[i].scheme;
      const int nfld = (sc == FFTC_EM_SUB ? 3 : (sc == FFTC_BASIC_SUB ? 2 : 1)) +
                       ((sc == FFTC_EM || sc == FFTC_EM_SUB) ? 2 : 1);
      per = std::max(per, (size_t)nfld * sizeof(double2) * (size_t)pb->d * (size_t)N + (size_t)N + (32u << 20));
    }
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess && per > 0)
      width = std::max(1, std::min<int>(width, (int)std::min<size_t>((size_t)(0.85 * (double)fr) / per, 64)));
  }
  if (width <= 1) {
    for (int32_t i = 0; i < n_points; ++i) {
      int rc = fftc_solve(pb, &params[i], histories + (size_t)i * history_cap * 3, history_cap, nullptr, nullptr,
                          nullptr, &out[i], stream);
      if (rc) {
        g_err = "point " + std::to_string(i) + ": " + g_err;
        return rc;
      }
    }
    return 0;
  }
  int dev = 0;
  CK(cudaGetDevice(&dev));
  cudaEvent_t ready;
  CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  CK(cudaEventRecord(ready, (cudaStream_t)stream));  // chi and friends are ordered on the caller's stream
  std::atomic<int32_t> next{0};
  std::atomic<int> first_bad{-1};
  std::vector<int> rcs(n_points, 0);
  std::vector<std::string> errs(n_points);
  auto worker = [&]() {
    cudaSetDevice(dev);
    cudaStream_t ws = nullptr;
    if (cudaStreamCreateWithFlags(&ws, cudaStreamNonBlocking) != cudaSuccess) {
      first_bad = 0;
      return;
    }
    cudaStreamWaitEvent(ws, ready, 0);
    for (int32_t i; first_bad.load() < 0 && (i = next.fetch_add(1)) < n_points;) {
      rcs[i] = fftc_solve(pb, &params[i], histories + (size_t)i * history_cap * 3, history_cap, nullptr, nullptr,
                          nullptr, &out[i], ws);
      if (rcs[i]) {
        errs[i] = g_err;
        int expect = -1;
        first_bad.compare_exchange_strong(expect, i);
      }
    }
    cudaStreamSynchronize(ws);
    cudaStreamDestroy(ws);
  };
  std::vector<std::thread> pool;
  for (int w = 0; w < width; ++w) pool.emplace_back(worker);
  for (auto& t : pool) t.join();
  cudaEventDestroy(ready);
  const int bad = first_bad.load();
  if (bad >= 0) {
    g_err = "point " + std::to_string(bad) + ": " + (errs[bad].empty() ? "stream setup failed" : errs[bad]);
    return rcs[bad] ? rcs[bad] : 1;
  }
  return 0;
}

// ---------------------------------------------------------------------------
// z-slab decomposition (BASELINE config 4): one rank per GPU owns z-planes
// [z0, z0 + nzl) of the state and work fields; the z pass runs on a y-slab
// copy [y0, y0 + nyl) produced by the caller's all-to-all transpose.  Every
// reduction leaves a rank-local partial that the caller all-reduces.
// ---------------------------------------------------------------------------
struct fftc_slab {
  Args row;     // z-slab geometry (local nz), work fields A_z / B_z
  Args mid;     // y-slab geometry (global nz), work fields A_y / B_y
  ColGeom yf{}, zg{};
  int scheme = 0, lgx = 0, lgy = 0, lgz = 0;
  bool em_type = false;
  long long N_l = 0;
  char* ws = nullptr;
  double* tot_dev = nullptr;  // 8 doubles of host-supplied totals
  DevState* hst = nullptr;
  Col3Pass yfwd3, yinv3, mid3;  // TMA tile column passes where the lengths allow
  long long z0 = 0, nyl = 0;    // this rank's first z-plane and y-slab height
  bool fused = false;           // transposes fused into the y forward / z passes (fftc_slab_set_peers)
  PeerOut* po_dev = nullptr;    // [0]: y forward -> y-slabs, [1]: z pass -> z-slabs
};

int fftc_slab_create(const fftc_slab_desc* sd, const fftc_params* pr, void* Az, void* Bz, void* Ay, void* By,
                     fftc_slab** out, void* stream) {
  g_err.clear();
  if (!sd || !pr || !out || sd->d != 3) {
    g_err = "slab: d must be 3";
    return 2;
  }
  const long long nx = sd->n[0], ny = sd->n[1], nz = sd->n[2];
  const int lgx = lg2_exact(nx), lgy = lg2_exact(ny), lgz = lg2_exact(nz);
  if (lgx < 0 || lgy < 0 || lgz < 0 || sd->nzl < 1 || sd->nyl < 1 || sd->nzl * ny != sd->nyl * nz) {
    g_err = "slab: unsupported grid or inconsistent slabs";
    return 3;
  }
  if (ensure_registry()) return 1;
  Registry& R = reg();
  cudaStream_t s = (cudaStream_t)stream;
  fftc_slab* sl = new fftc_slab();
  const int d = 3;
  const long long N_l = nx * ny * sd->nzl, N_g = nx * ny * nz;
  sl->N_l = N_l;
  sl->scheme = pr->scheme;
  sl->lgx = lgx;
  sl->lgy = lgy;
  sl->lgz = lgz;
  sl->em_type = (pr->scheme == FFTC_EM || pr->scheme == FFTC_EM_SUB);
  Args& a = sl->row;
  memset(&a, 0, sizeof(a));
  a.d = d;
  a.nx = (int)nx;
  a.ny = (int)ny;
  a.nz = (int)sd->nzl;
  a.N = N_l;
  a.chi = sd->chi;
  a.row_e = row_e((int)nx, (int)pr->scheme);
  fill_scalars(a, pr, d, N_g);  // means and normalisations are global
  a.dist = 1;
  const int nslots = pr->scheme == FFTC_EM_SUB ? 3 : (pr->scheme == FFTC_BASIC_SUB ? 2 : 1);
  const size_t fld = sizeof(double2) * (size_t)d * N_l;
  // a ring: fftc_slab_monitor hands every record to the caller as it is written
  const int hist_cap = 1024;
  const size_t pc = (size_t)R.num_sms * 64 * NQMAX + 16 * NQMAX;
  const size_t bytes = fld * nslots + sizeof(double) * pc + sizeof(double) * 3 * hist_cap + sizeof(DevState) +
                       sizeof(int2) * (size_t)ny * sd->nzl + sizeof(double) * 8 + (size_t)N_l + 256 + 8192;
  if (cudaMalloc((void**)&sl->ws, bytes) != cudaSuccess) {
    g_err = "slab: workspace allocation failed";
    delete sl;
    return 1;
  }
  size_t o = 0;
  auto carve = [&](size_t b) {
    char* p = sl->ws + o;
    o += (b + 255) & ~(size_t)255;
    return p;
  };
  for (int i = 0; i < nslots; ++i) a.X[i] = (double2*)carve(fld);
  a.partials = (double*)carve(sizeof(double) * pc);
  a.history = (double*)carve(sizeof(double) * 3 * hist_cap);
  a.hist_cap = hist_cap;
  a.st = (DevState*)carve(sizeof(DevState));
  a.row_ext = (const int2*)carve(sizeof(int2) * (size_t)ny * sd->nzl);
  a.chiT = nx >= 16 ? (const uint8_t*)carve((size_t)N_l) : nullptr;  // thread-blocked chi rows (TMA row sweeps)
  sl->tot_dev = (double*)carve(sizeof(double) * 8);
  a.A = (double2*)Az;
  a.B = sl->em_type ? (double2*)Bz : (double2*)Az;
  a.tw[0] = R.tw[lgx];
  a.tw[1] = R.tw[lgy];
  a.tw[2] = R.tw[lgz];
  sl->mid = a;
  sl->mid.nz = (int)nz;  // the z pass sees whole z lines
  sl->z0 = sd->z0;
  sl->nyl = sd->nyl;
  sl->mid.A = (double2*)Ay;
  sl->mid.B = sl->em_type ? (double2*)By : (double2*)Ay;
  // y passes on the z-slab (lines along y, one per (z, x-strip, component))
  sl->yf.axis = 1;
  sl->yf.nouter = (int)sd->nzl;
  sl->yf.stride = nx;
  sl->yf.ostride = nx * ny;
  sl->yf.nstrips = (int)(nx / 2);
  // z pass on the y-slab, layout (c, y_l, z, x): lines along z, stride nx
  sl->zg.axis = 2;
  sl->zg.nouter = (int)sd->nyl;
  sl->zg.stride = nx;
  sl->zg.ostride = nz * nx;
  sl->zg.nstrips = (int)(nx / R.tab[lgz].col3_w);
  sl->zg.o0 = (int)sd->y0;
  sl->zg.on = (int)ny;
  {
    const LTable& TY = R.tab[lgy];
    const LTable& TZ = R.tab[lgz];
    const int nf = sl->em_type ? 2 : 1;
    col3_pass(sl->yfwd3, TY.col[KC_FWD3T], a, Az, sl->em_type ? Bz : nullptr, ny, nx, sd->nzl, nx * ny, N_l, nf, 1,
              0, (int)sd->nzl);
    col3_pass(sl->yinv3, TY.col[KC_INV3T], a, Az, nullptr, ny, nx, sd->nzl, nx * ny, N_l, 1, 1, 0, (int)sd->nzl);
    col3_pass(sl->mid3, TZ.col[sl->em_type ? KC_MID3T_EM : KC_MID3T_BASIC], sl->mid, Ay, sl->em_type ? By : nullptr,
              nz, nx, sd->nyl, nz * nx, sd->nyl * nz * nx, nf, 2, (int)sd->y0, (int)ny);
  }
  if (cudaMallocHost((void**)&sl->hst, sizeof(DevState)) != cudaSuccess ||
      cudaMemsetAsync(a.st, 0, sizeof(DevState), s) != cudaSuccess) {
    g_err = "slab: state allocation failed";
    cudaFree(sl->ws);
    delete sl;
    return 1;
  }
  *out = sl;
  return 0;
}

static int slab_read_state(fftc_slab* sl, cudaStream_t s) {
  CK(cudaMemcpyAsync(sl->hst, sl->row.st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return 0;
}

int fftc_slab_phase(fftc_slab* sl, int32_t phase, double* out, void* stream) {
  g_err.clear();
  Registry& R = reg();
  cudaStream_t s = (cudaStream_t)stream;
  Launcher Lc(s, R.num_sms);
  Args& a = sl->row;
  const int d = a.d;
  const LTable& TX = R.tab[sl->lgx];
  const LTable& TY = R.tab[sl->lgy];
  const LTable& TZ = R.tab[sl->lgz];
  const long long rows = (long long)a.ny * a.nz;
  const long long yf_lines = (long long)sl->yf.nouter * sl->yf.nstrips * d;
  int rc = 0;
  void* a1[] = {&a};
  switch (phase) {
    case FFTC_SLAB_INIT: {
      CK(cudaMemsetAsync(a.st, 0, sizeof(DevState), s));
      unsigned g = (unsigned)std::min<long long>((rows + 7) / 8, (long long)R.num_sms * 8);
      void* ea[] = {(void*)&a.chi, (void*)&a.nx, (void*)&rows, (void*)&a.row_ext};
      if ((rc = Lc.raw((const void*)k_row_extent, g, 256, 0, ea, K_INIT))) return rc;
      if (a.chiT) {
        const long long chunks = rows * (a.nx / a.row_e);
        unsigned gp = (unsigned)std::min<long long>((chunks + 255) / 256, (long long)R.num_sms * 16);
        void* pa[] = {(void*)&a.chi, (void*)&a.nx, (void*)&rows, (void*)&a.chiT, (void*)&a.row_e};
        if ((rc = Lc.raw((const void*)k_chi_perm16, gp, 256, 0, pa, K_INIT))) return rc;
      }
      switch (sl->scheme) {
        case FFTC_BASIC: rc = launch_elementwise(k_init<BASIC>, Lc, (long long)d * a.N, a, K_INIT); break;
        case FFTC_EM: rc = launch_elementwise(k_init<EM>, Lc, (long long)d * a.N, a, K_INIT); break;
        case FFTC_BASIC_SUB: rc = launch_elementwise(k_init<BASIC_SUB>, Lc, (long long)d * a.N, a, K_INIT); break;
        default: rc = launch_elementwise(k_init<EM_SUB>, Lc, (long long)d * a.N, a, K_INIT); break;
      }
      if (rc) return rc;
      if (slab_read_state(sl, s)) return 1;
      for (int c = 0; c < 3; ++c) {
        out[2 * c] = sl->hst->delta[c].x;
        out[2 * c + 1] = sl->hst->delta[c].y;
      }
      return 0;
    }
    case FFTC_SLAB_ROWS_FWD: {
      if ((rc = Lc.go(TX.s1[sl->scheme], (long long)d * rows, a1, K_SWEEP1))) return rc;
      if (sl->fused) {
        // y forward with its output rows written straight into the owning
        // ranks' y-slabs: this pass IS the forward transpose
        const PeerOut* po = sl->po_dev;
        void* ay[] = {&a, &sl->yfwd3.g, &sl->yfwd3.mA, &sl->yfwd3.mB, &po};
        if ((rc = Lc.go(TY.col[KC_FWD3P], sl->yfwd3.tiles, ay, K_YFWD))) return rc;
      } else if (sl->yfwd3.ok) {
        const PeerOut* no_peer = nullptr;
        void* ay[] = {&a, &sl->yfwd3.g, &sl->yfwd3.mA, &sl->yfwd3.mB, &no_peer};
        if ((rc = Lc.go(*sl->yfwd3.k, sl->yfwd3.tiles, ay, K_YFWD))) return rc;
      } else {
        void* ayf[] = {&a, &sl->yf};
        if ((rc = Lc.go(TY.col[KC_FWD], yf_lines, ayf, K_YFWD))) return rc;
        if (sl->em_type) {
          Args aB = a;
          aB.A = a.B;
          void* ab[] = {&aB, &sl->yf};
          if ((rc = Lc.go(TY.col[KC_FWD], yf_lines, ab, K_YFWD))) return rc;
        }
      }
      if (slab_read_state(sl, s)) return 1;
      for (int c = 0; c < 3; ++c) {
        out[2 * c] = sl->hst->jmean[c].x;
        out[2 * c + 1] = sl->hst->jmean[c].y;
      }
      out[6] = sl->hst->js2;
      return 0;
    }
    case FFTC_SLAB_MID: {
      if (sl->fused) {
        // z pass writing back into the owning ranks' z-slabs: the backward transpose
        const PeerOut* po = sl->po_dev + 1;
        void* am[] = {&sl->mid, &sl->mid3.g, &sl->mid3.mA, &sl->mid3.mB, &po};
        if ((rc = Lc.go(TZ.col[sl->em_type ? KC_MID3P_EM : KC_MID3P_BASIC], sl->mid3.tiles, am, K_MID))) return rc;
      } else if (sl->mid3.ok) {
        const PeerOut* no_peer = nullptr;
        void* am[] = {&sl->mid, &sl->mid3.g, &sl->mid3.mA, &sl->mid3.mB, &no_peer};
        if ((rc = Lc.go(*sl->mid3.k, sl->mid3.tiles, am, K_MID))) return rc;
      } else {
        const KInfo& k = TZ.col[sl->em_type ? KC_MID3_EM : KC_MID3_BASIC];
        void* am[] = {&sl->mid, &sl->zg};
        const long long lines = (long long)sl->zg.nouter * sl->zg.nstrips * (sl->em_type ? 2 : 1);
        if ((rc = Lc.go(k, lines, am, K_MID))) return rc;
      }
      if (slab_read_state(sl, s)) return 1;
      out[0] = sl->hst->parseval;
      return 0;
    }
    case FFTC_SLAB_ROWS_INV: {
      if (sl->yinv3.ok) {
        const PeerOut* no_peer = nullptr;
        void* ay[] = {&a, &sl->yinv3.g, &sl->yinv3.mA, &sl->yinv3.mB, &no_peer};
        if ((rc = Lc.go(*sl->yinv3.k, sl->yinv3.tiles, ay, K_YINV))) return rc;
      } else {
        void* ai[] = {&a, &sl->yf};
        if ((rc = Lc.go(TY.col[KC_INV], yf_lines, ai, K_YINV))) return rc;
      }
      if ((rc = Lc.go(TX.s3[sl->scheme], (long long)d * rows, a1, K_SWEEP3))) return rc;
      if (slab_read_state(sl, s)) return 1;
      for (int c = 0; c < 3; ++c) {
        out[2 * c] = sl->hst->delta[c].x;
        out[2 * c + 1] = sl->hst->delta[c].y;
      }
      return 0;
    }
    default:
      g_err = "slab: bad phase";
      return 2;
  }
}

int fftc_slab_set_delta(fftc_slab* sl, const double* delta6, void* stream) {
  g_err.clear();
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaMemcpyAsync(sl->tot_dev, delta6, sizeof(double) * 6, cudaMemcpyHostToDevice, s));
  const double* dp = sl->tot_dev;
  void* args[] = {&sl->row, &dp};
  CK(cudaLaunchKernel((const void*)k_dist_set_delta, dim3(1), dim3(32), args, 0, s));
  CK(cudaStreamSynchronize(s));
  return 0;
}

int fftc_slab_monitor(fftc_slab* sl, const double* totals8, double* rec, void* stream) {
  g_err.clear();
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaMemcpyAsync(sl->tot_dev, totals8, sizeof(double) * 8, cudaMemcpyHostToDevice, s));
  const double* tp = sl->tot_dev;
  void* args[] = {&sl->row, &tp};
  CK(cudaLaunchKernel((const void*)k_dist_monitor, dim3(1), dim3(32), args, 0, s));
  if (slab_read_state(sl, s)) return 1;
  DevState* h = sl->hst;
  rec[0] = h->stopped;
  rec[1] = h->status;
  rec[2] = h->degenerate;
  rec[3] = h->nrec;
  rec[4] = h->last_sstar.x;
  rec[5] = h->last_sstar.y;
  rec[6] = 0.0;
  if (h->nrec > 0) {
    double r3[3];
    const long long slot = (h->nrec - 1) % sl->row.hist_cap;
    CK(cudaMemcpy(r3, sl->row.history + 3 * slot, sizeof(r3), cudaMemcpyDeviceToHost));
    rec[4] = r3[0];
    rec[5] = r3[1];
    rec[6] = r3[2];
  }
  return 0;
}

int fftc_slab_finalize(fftc_slab* sl, void* E, void* J, void* aug, double* means12, void* stream) {
  g_err.clear();
  Registry& R = reg();
  cudaStream_t s = (cudaStream_t)stream;
  Launcher Lc(s, R.num_sms);
  Args a = sl->row;
  a.outE = (double2*)E;
  a.outJ = (double2*)J;
  a.outAug = (double2*)aug;
  int rc;
  switch (sl->scheme) {
    case FFTC_BASIC: rc = launch_elementwise(k_finalize<BASIC>, Lc, (long long)a.d * a.N, a, K_FINAL); break;
    case FFTC_EM: rc = launch_elementwise(k_finalize<EM>, Lc, (long long)a.d * a.N, a, K_FINAL); break;
    case FFTC_BASIC_SUB: rc = launch_elementwise(k_finalize<BASIC_SUB>, Lc, (long long)a.d * a.N, a, K_FINAL); break;
    default: rc = launch_elementwise(k_finalize<EM_SUB>, Lc, (long long)a.d * a.N, a, K_FINAL); break;
  }
  if (rc) return rc;
  if (slab_read_state(sl, s)) return 1;
  for (int c = 0; c < 3; ++c) {
    means12[2 * c] = sl->hst->meanE[c].x;
    means12[2 * c + 1] = sl->hst->meanE[c].y;
    means12[6 + 2 * c] = sl->hst->meanJ[c].x;
    means12[6 + 2 * c + 1] = sl->hst->meanJ[c].y;
  }
  return 0;
}

int fftc_slab_set_peers(fftc_slab* sl, int32_t world, void* const* Ay, void* const* By, void* const* Az,
                        void* stream) {
  g_err.clear();
  if (!sl || !Ay || !Az || world < 1 || world > 8 || (sl->em_type && !By)) {
    g_err = "slab peers: null argument or world outside 1..8";
    return 2;
  }
  const Args& a = sl->row;
  const long long nx = a.nx, ny = a.ny, nzl = a.nz, nz = sl->mid.nz, nyl = sl->nyl;
  if (ny % world || nz % world || ny / world != nyl || nz / world != nzl) {
    g_err = "slab peers: world does not match the slab geometry";
    return 2;
  }
  Registry& R = reg();
  const bool kernels = R.tab[sl->lgy].col[KC_FWD3P].max_active > 0 &&
                       R.tab[sl->lgz].col[sl->em_type ? KC_MID3P_EM : KC_MID3P_BASIC].max_active > 0;
  if (!sl->yfwd3.ok || !sl->mid3.ok || !kernels) {
    g_err = "slab peers: fused transposes need y and z lines of 256..1024 (TMA tile passes)";
    return 3;
  }
  // z-blocked slabs for the fused mode: the z-slab work fields (rows of the
  // row sweeps, y lines of the y passes, targets of the z pass's stores) and
  // the y-slabs (targets of the y forward pass's stores, z lines of the z
  // pass) keep 2^zs planes of a row adjacent, as the monolithic solve does,
  // so neither the transposing stores nor the z lines land one 2 MB page per
  // 32 bytes.  Falls back to the plain layouts when a map does not encode.
  int zsA = zblock_shift(nx, ny, nzl), zsY = zblock_shift(nx, nyl, nz);
  {
    Registry& RR = reg();
    const LTable& TY = RR.tab[sl->lgy];
    const LTable& TZ = RR.tab[sl->lgz];
    const int nf = sl->em_type ? 2 : 1;
    Col3Pass yf, yi, md;
    Args ay = sl->mid;
    ay.ny = (int)nyl;  // the y-slab holds nyl rows of every z plane
    bool ok = zsA > 0 && zsY > 0 &&
              col3_pass_zblk(yf, TY.col[KC_FWD3T], a, a.A, sl->em_type ? a.B : nullptr, 1, zsA, nf) &&
              col3_pass_zblk(yi, TY.col[KC_INV3T], a, a.A, nullptr, 1, zsA, 1) &&
              col3_pass_zblk(md, TZ.col[sl->em_type ? KC_MID3T_EM : KC_MID3T_BASIC], ay, sl->mid.A,
                             sl->em_type ? sl->mid.B : nullptr, 2, zsY, nf);
    if (ok) {
      md.g.o0 = sl->zg.o0;  // global y of the slab's first row (wave numbers)
      md.g.on = (int)ny;
      sl->yfwd3 = yf;
      sl->yinv3 = yi;
      sl->mid3 = md;
      sl->row.zbs = zsA;
    } else {
      zsA = zsY = 0;
    }
  }
  PeerOut po[2];
  memset(po, 0, sizeof(po));
  for (int q = 0; q < world; ++q) {
    po[0].dst[0][q] = (double2*)Ay[q];  // y forward -> y-slab (c, y_l, z, x) of rank q
    po[0].dst[1][q] = (double2*)(sl->em_type ? By[q] : Ay[q]);
    po[1].dst[0][q] = (double2*)Az[q];  // z pass -> z-slab (c, z_l, y, x) of rank q
    po[1].dst[1][q] = (double2*)Az[q];
  }
  po[0].world = po[1].world = world;
  po[0].rows_per_rank = (int)nyl;
  po[0].line_stride = nz * nx;  // y_l
  po[0].outer_stride = nx;      // z
  po[0].outer0 = sl->z0;        // z of this rank's plane z_l
  po[0].comp_stride = nyl * nz * nx;
  po[1].rows_per_rank = (int)nzl;
  po[1].line_stride = ny * nx;  // z_l
  po[1].outer_stride = nx;      // y
  po[1].outer0 = sl->zg.o0;     // y0
  po[1].comp_stride = nzl * ny * nx;
  po[0].zs = zsY;  // y-slab rows: z blocked, the line (y) inside the block row
  po[0].blk_line = 0;
  po[0].bn = nyl;
  po[0].row_len = nx;
  po[1].zs = zsA;  // z-slab rows: the line (z) blocked
  po[1].blk_line = 1;
  po[1].bn = ny;
  po[1].row_len = nx;
  cudaStream_t s = (cudaStream_t)stream;
  if (!sl->po_dev) CK(cudaMalloc((void**)&sl->po_dev, sizeof(po)));
  CK(cudaMemcpyAsync(sl->po_dev, po, sizeof(po), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  sl->fused = true;
  return 0;
}

int fftc_ipc_alloc(int64_t bytes, void** ptr) {
  g_err.clear();
  if (!ptr || bytes <= 0) {
    g_err = "ipc alloc: bad argument";
    return 2;
  }
  CK(cudaMalloc(ptr, (size_t)bytes));  // a whole allocation: its IPC handle maps exactly this buffer
  return 0;
}
int fftc_ipc_free(void* ptr) {
  g_err.clear();
  CK(cudaFree(ptr));
  return 0;
}
int fftc_ipc_handle(void* ptr, void* handle64) {
  g_err.clear();
  if (!ptr || !handle64) {
    g_err = "ipc handle: null argument";
    return 2;
  }
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, ptr));
  static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
  memcpy(handle64, &h, sizeof(h));
  return 0;
}
int fftc_ipc_open(const void* handle64, void** ptr) {
  g_err.clear();
  if (!handle64 || !ptr) {
    g_err = "ipc open: null argument";
    return 2;
  }
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  CK(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return 0;
}
int fftc_ipc_close(void* ptr) {
  g_err.clear();
  CK(cudaIpcCloseMemHandle(ptr));
  return 0;
}

void fftc_slab_destroy(fftc_slab* sl) {
  if (!sl) return;
  cudaDeviceSynchronize();
  if (sl->po_dev) cudaFree(sl->po_dev);
  if (sl->ws) cudaFree(sl->ws);
  if (sl->hst) cudaFreeHost(sl->hst);
  delete sl;
}

int fftc_solve_host(const fftc_problem* pb, const fftc_params* pr, double* history, int64_t history_cap,
                    void* E_host, void* J_host, void* aug_host, fftc_result* out) {
  g_err.clear();
  if (!pb || !pb->chi) {
    g_err = "null problem";
    return 2;
  }
  const long long N = pb->n[0] * pb->n[1] * (pb->d == 3 ? pb->n[2] : 1);
  const size_t fld = sizeof(double2) * (size_t)pb->d * N;
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  uint8_t* chi = nullptr;
  void *E = nullptr, *J = nullptr, *aug = nullptr;
  int rc = 0;
  do {
    if (cudaMallocAsync((void**)&chi, N, s) != cudaSuccess) { rc = 1; break; }
    if (cudaMemcpyAsync(chi, pb->chi, N, cudaMemcpyHostToDevice, s) != cudaSuccess) { rc = 1; break; }
    if (E_host && cudaMallocAsync(&E, fld, s) != cudaSuccess) { rc = 1; break; }
    if (J_host && cudaMallocAsync(&J, fld, s) != cudaSuccess) { rc = 1; break; }
    if (aug_host && cudaMallocAsync(&aug, 3 * fld, s) != cudaSuccess) { rc = 1; break; }
    fftc_problem p2 = *pb;
    p2.chi = chi;
    rc = fftc_solve(&p2, pr, history, history_cap, E, J, aug, out, s);
    if (rc) break;
    if (E_host && cudaMemcpyAsync(E_host, E, fld, cudaMemcpyDeviceToHost, s) != cudaSuccess) { rc = 1; break; }
    if (J_host && cudaMemcpyAsync(J_host, J, fld, cudaMemcpyDeviceToHost, s) != cudaSuccess) { rc = 1; break; }
    if (aug_host && cudaMemcpyAsync(aug_host, aug, 3 * fld, cudaMemcpyDeviceToHost, s) != cudaSuccess) { rc = 1; break; }
    if (cudaStreamSynchronize(s) != cudaSuccess) { rc = 1; break; }
  } while (0);
  if (rc == 1 && g_err.empty()) g_err = cudaGetErrorString(cudaGetLastError());
  if (chi) cudaFreeAsync(chi, s);
  if (E) cudaFreeAsync(E, s);
  if (J) cudaFreeAsync(J, s);
  if (aug) cudaFreeAsync(aug, s);
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  return rc;
}

}  // extern "C"

namespace fftc {
void set_last_error(const std::string& msg) { g_err = msg; }
void clear_last_error() { g_err.clear(); }
void add_launches(long long n) { g_launches += n; }
int device_sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) return 148;
  return n;
}
}  // namespace fftc

