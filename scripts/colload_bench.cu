// colload_bench.cu -- load-only microbenchmark for the 2-D column sweep's data
// movement: how fast can 148 SMs pull x-columns of a (2, L, L) complex128
// field out of HBM as TMA tensor boxes of W adjacent columns (16*W-byte box
// rows), with NSLOT boxes in flight per CTA, versus plain LDG.128 loads with
// W columns per warp instruction.  Nothing is computed; each thread touches
// one landed value so the slot is really consumed.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 colload_bench.cu -o colload_bench
//   ./colload_bench            (prints one line per variant)
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) {                                                            \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                          \
    }                                                                                   \
  } while (0)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NSLOT>
__global__ void __launch_bounds__(512, 1) k_tma(const __grid_constant__ CUtensorMap tm, int nlines, int W, int ncomp,
                                                 unsigned slot_bytes, int comp_per_box, double* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bars[NSLOT];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < NSLOT; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bars[s])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // a "line" = one box: W columns x L rows x comp_per_box components
  const int nmine = blockIdx.x < nlines ? (nlines - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int boxes_per_cgroup = nlines / (ncomp / comp_per_box);
  auto issue = [&](int k, int s) {
    const int line = blockIdx.x + k * gridDim.x;
    const int cg = line / boxes_per_cgroup, xb = line % boxes_per_cgroup;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bars[s])), "r"(slot_bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5}], [%6];" ::"r"(su(sm + (size_t)s * slot_bytes)),
        "l"(&tm), "r"(2 * W * xb), "r"(0), "r"(0), "r"(cg * comp_per_box), "r"(su(&bars[s]))
        : "memory");
  };
  if (tid == 0)
    for (int s = 0; s < NSLOT && s < nmine; ++s) issue(s, s);
  double acc = 0.0;
  for (int k = 0; k < nmine; ++k) {
    const int s = k % NSLOT;
    const unsigned par = (unsigned)((k / NSLOT) & 1);
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            su(&bars[s])),
        "r"(par)
        : "memory");
    const double* d = reinterpret_cast<const double*>(sm + (size_t)s * slot_bytes);
    for (unsigned i = tid; i < slot_bytes / 8; i += 8 * blockDim.x) acc += d[i];
    __syncthreads();
    if (tid == 0 && k + NSLOT < nmine) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(k + NSLOT, s);
    }
  }
  if (acc == 12345.678) sink[0] = acc;
}

template <int NSLOT>
__global__ void __launch_bounds__(512, 1) k_tma5(const __grid_constant__ CUtensorMap tm, int nlines, unsigned slot_bytes,
                                                  double* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bars[NSLOT];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < NSLOT; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bars[s])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nmine = blockIdx.x < nlines ? (nlines - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto issue = [&](int k, int s) {
    const int x = blockIdx.x + k * gridDim.x;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bars[s])), "r"(slot_bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5, %6}], [%7];" ::"r"(su(sm + (size_t)s * slot_bytes)),
        "l"(&tm), "r"(0), "r"(x), "r"(0), "r"(0), "r"(0), "r"(su(&bars[s]))
        : "memory");
  };
  if (tid == 0)
    for (int s = 0; s < NSLOT && s < nmine; ++s) issue(s, s);
  double acc = 0.0;
  for (int k = 0; k < nmine; ++k) {
    const int s = k % NSLOT;
    const unsigned par = (unsigned)((k / NSLOT) & 1);
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            su(&bars[s])),
        "r"(par)
        : "memory");
    const double* d = reinterpret_cast<const double*>(sm + (size_t)s * slot_bytes);
    for (unsigned i = tid; i < slot_bytes / 8; i += 8 * blockDim.x) acc += d[i];
    __syncthreads();
    if (tid == 0 && k + NSLOT < nmine) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(k + NSLOT, s);
    }
  }
  if (acc == 12345.678) sink[0] = acc;
}

// LDG: a CTA of 512 threads reads lines of W columns x L rows x 2 comps
// straight into registers (16 LDG.128 per thread per pass), lane bits
// [log2 W) = column so one warp instruction covers 32/W rows x 16W bytes
__global__ void __launch_bounds__(512, 1) k_ldg(const double2* __restrict__ f, int L, int W, int ncomp, double* sink) {
  const int tid = threadIdx.x;
  const int nlines = (L / W);
  const int per_pass = 512 / W;  // rows x comps covered by one pass
  double acc = 0.0;
  for (int line = blockIdx.x; line < nlines; line += gridDim.x) {
    const int x = line * W + (tid % W);
    const int r0 = tid / W;
    double2 v[16];
    for (int base = 0; base < L * ncomp; base += per_pass * 16) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int rc = base + r0 + i * per_pass;
        const int c = rc / L, y = rc % L;
        v[i] = __ldg(&f[(size_t)c * L * L + (size_t)y * L + x]);
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) acc += v[i].x;
    }
  }
  if (acc == 12345.678) sink[0] = acc;
}

int main() {
  const int L = 2048, NC = 2;
  double2* f;
  double* sink;
  const size_t bytes = (size_t)NC * L * L * sizeof(double2);
  CK(cudaMalloc(&f, bytes));
  CK(cudaMalloc(&sink, 8));
  CK(cudaMemset(f, 0, bytes));
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  EncodeTiledFn enc = (EncodeTiledFn)p;
  int nsm;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  printf("field %.0f MB (2 comps x %d^2 complex128), %d SMs\n", bytes / 1e6, L, nsm);

  struct V {
    int W, rows_per_box_blocks, comp_per_box, nslot;
  };
  // rows_per_box_blocks: the box covers 256 x this many rows (8 = whole line)
  const V vs[] = {{1, 8, 2, 1}, {1, 8, 2, 2}, {1, 8, 2, 3}, {2, 8, 1, 1}, {2, 8, 1, 2}, {2, 8, 1, 3},
                  {4, 4, 1, 3}, {4, 8, 1, 1}, {8, 2, 1, 3}, {8, 4, 1, 1}, {16, 1, 1, 3}, {16, 2, 1, 3},
                  {1, 4, 1, 3}, {2, 4, 1, 3}, {1, 8, 1, 3}, {4, 2, 1, 3}};
  for (const V& v : vs) {
    CUtensorMap tm;
    cuuint64_t dims[4] = {(cuuint64_t)(2 * L), 256, (cuuint64_t)(L / 256), (cuuint64_t)NC};
    cuuint64_t strides[3] = {(cuuint64_t)L * 16, (cuuint64_t)L * 16 * 256, (cuuint64_t)L * L * 16};
    cuuint32_t box[4] = {(cuuint32_t)(2 * v.W), 256, (cuuint32_t)v.rows_per_box_blocks, (cuuint32_t)v.comp_per_box};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, f, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("encode failed W=%d\n", v.W);
      continue;
    }
    const unsigned slot = (unsigned)(16 * v.W * 256 * v.rows_per_box_blocks * v.comp_per_box);
    const size_t smem = (size_t)slot * v.nslot;
    if (smem > 227 * 1024) {
      printf("W=%d slots=%d: %zu B smem too big\n", v.W, v.nslot, smem);
      continue;
    }
    // boxes: column groups x row groups x comp groups; row groups only via multiple "lines" along blocks
    // (for rows_per_box_blocks < 8 we just read the first part of every column: scale bytes accordingly)
    const int nlines = (L / v.W) * (NC / v.comp_per_box);
    auto launch = [&](int ns) {
      if (ns == 1) {
        cudaFuncSetAttribute(k_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_tma<1><<<nsm, 512, smem>>>(tm, nlines, v.W, NC, slot, v.comp_per_box, sink);
      } else if (ns == 2) {
        cudaFuncSetAttribute(k_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_tma<2><<<nsm, 512, smem>>>(tm, nlines, v.W, NC, slot, v.comp_per_box, sink);
      } else {
        cudaFuncSetAttribute(k_tma<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_tma<3><<<nsm, 512, smem>>>(tm, nlines, v.W, NC, slot, v.comp_per_box, sink);
      }
    };
    for (int i = 0; i < 3; ++i) launch(v.nslot);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    const int reps = 10;
    for (int i = 0; i < reps; ++i) launch(v.nslot);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double moved = (double)nlines * slot;
    printf("TMA  W=%2d (box rows %3d B) rows/box=%4d comps/box=%d nslot=%d slot=%6u B: %7.1f us  %7.0f GB/s  %.3f box-rows/clk/SM\n",
           v.W, 16 * v.W, 256 * v.rows_per_box_blocks, v.comp_per_box, v.nslot, slot, 1e3 * ms / reps,
           moved / (1e6 * ms / reps), (double)nlines * 256 * v.rows_per_box_blocks * v.comp_per_box /
                                           (1e-3 * ms / reps * 1.9e9 * nsm));
  }
  // row-pair interleaved field: element (c, y, x) at c*L*L + ((y>>1)*L + x)*2 + (y&1); a column's box is
  // {4 doubles = rows 2m, 2m+1} x {1 x} x {128 pairs} x {8 pair blocks} x {comps}: 32-byte rows
  for (int ns : {1, 2, 3}) {
    CUtensorMap tm;
    const int lo = 128, hi = L / 2 / lo;
    cuuint64_t dims[5] = {4, (cuuint64_t)L, (cuuint64_t)lo, (cuuint64_t)hi, (cuuint64_t)NC};
    cuuint64_t strides[4] = {32, (cuuint64_t)32 * L, (cuuint64_t)32 * L * lo, (cuuint64_t)16 * L * L};
    cuuint32_t box[5] = {4, 1, (cuuint32_t)lo, (cuuint32_t)hi, 2};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, f, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("pair map encode failed %d\n", (int)r); break; }
    const unsigned slot = (unsigned)(2 * L * 16);
    const size_t smem = (size_t)slot * ns;
    const int nlines = L;
    auto launch = [&]() {
      if (ns == 1) { cudaFuncSetAttribute(k_tma5<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                     k_tma5<1><<<nsm, 512, smem>>>(tm, nlines, slot, sink); }
      else if (ns == 2) { cudaFuncSetAttribute(k_tma5<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                     k_tma5<2><<<nsm, 512, smem>>>(tm, nlines, slot, sink); }
      else { cudaFuncSetAttribute(k_tma5<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                     k_tma5<3><<<nsm, 512, smem>>>(tm, nlines, slot, sink); }
    };
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int i = 0; i < 10; ++i) launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("PAIR (32-B rows, 1 column x 2 comps per box) nslot=%d: %7.1f us  %7.0f GB/s\n", ns, 1e3 * ms / 10,
           (double)nlines * slot / (1e6 * ms / 10));
  }
  for (int W : {1, 2, 4, 8}) {
    for (int i = 0; i < 3; ++i) k_ldg<<<nsm * 2, 512>>>(f, L, W, NC, sink);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    const int reps = 10;
    for (int i = 0; i < reps; ++i) k_ldg<<<nsm * 2, 512>>>(f, L, W, NC, sink);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("LDG  W=%2d: %7.1f us  %7.0f GB/s\n", W, 1e3 * ms / reps, bytes / (1e6 * ms / reps));
  }
  return 0;
}
