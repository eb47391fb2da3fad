// zload_bench.cu -- load-only microbenchmark for the 3-D column passes at
// n^3 (default 1024^3, 3 components, complex128 = 48 GiB): TMA tiles of W
// adjacent x-columns x 3 components along y or z, in the reference layout
// (c, z, y, x) and in a z-blocked layout (c, z/ZB, y, z%ZB, x) that keeps ZB
// consecutive z-planes of one y-row adjacent (z-lines touch n/ZB 2 MB pages
// instead of n).  Each CTA keeps NSLOT tiles in flight; nothing is computed.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 zload_bench.cu -o zload_bench
//   ./zload_bench [n]
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

// line = (outer o, x-tile xt); coords {2*W*xt, 0, c2(o), c3(o), 0}
template <int NSLOT>
__global__ void __launch_bounds__(256, 1) k_tma(const __grid_constant__ CUtensorMap tm, int nlines, int ntiles,
                                                 int mode, int n, int zb, unsigned slot_bytes, double* sink) {
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
    const int line = blockIdx.x + k * gridDim.x;
    const int xt = line % ntiles, o = line / ntiles;
    int c1 = 0, c2 = 0, c3 = 0;
    if (mode == 0) {  // z-line, reference layout: dims {2n, 256, n/256, n(y), 3}; outer = y
      c3 = o;
    } else if (mode == 1) {  // z-line, blocked: dims {2n, zb, n/zb, n(y), 3}; outer = y
      c3 = o;
    } else if (mode == 2) {  // y-line, reference: dims {2n, 256, n/256, n(z), 3}; outer = z
      c3 = o;
    } else {  // y-line, blocked: dims {2n, 256, (n/256)*(n/zb), zb, 3}; outer = z = zh*zb + zl
      const int zh = o / zb, zl = o % zb;
      c2 = zh * (n / 256);
      c3 = zl;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bars[s])), "r"(slot_bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5, %6}], [%7];" ::"r"(su(sm + (size_t)s * slot_bytes)),
        "l"(&tm), "r"(xt * 0 + 2 * (int)(slot_bytes / (16 * 3 * n)) * xt), "r"(c1), "r"(c2), "r"(c3), "r"(0),
        "r"(su(&bars[s]))
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
    acc += d[tid * 8];
    __syncthreads();
    if (tid == 0 && k + NSLOT < nmine) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(k + NSLOT, s);
    }
  }
  if (acc == 12345.678) sink[0] = acc;
}

int main(int argc, char** argv) {
  const long long n = argc > 1 ? atoll(argv[1]) : 1024;
  const size_t bytes = (size_t)3 * n * n * n * 16;
  void* f;
  double* sink;
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
  printf("n=%lld field %.1f GB, %d SMs\n", n, bytes / 1e9, nsm);
  const unsigned long long N = n;
  for (int mode = 0; mode < 4; ++mode) {
    for (int zb : {8, 16, 32}) {
      if ((mode == 0 || mode == 2) && zb != 8) continue;
      for (int W : {2, 4}) {
        if (W * 3 * n * 16 * 2 > 220 * 1024) continue;
        CUtensorMap tm;
        cuuint64_t dims[5], strides[4];
        cuuint32_t box[5];
        const unsigned long long C = 3 * N * N * N * 16;  // comp stride bytes
        if (mode == 0) {
          dims[0] = 2 * N; dims[1] = 256; dims[2] = N / 256; dims[3] = N; dims[4] = 3;
          strides[0] = N * N * 16; strides[1] = N * N * 16 * 256; strides[2] = N * 16; strides[3] = C / 3;
          box[0] = 2 * W; box[1] = 256; box[2] = N / 256; box[3] = 1; box[4] = 3;
        } else if (mode == 1) {
          dims[0] = 2 * N; dims[1] = zb; dims[2] = N / zb; dims[3] = N; dims[4] = 3;
          strides[0] = N * 16; strides[1] = N * N * zb * 16; strides[2] = zb * N * 16; strides[3] = C / 3;
          box[0] = 2 * W; box[1] = zb; box[2] = N / zb; box[3] = 1; box[4] = 3;
        } else if (mode == 2) {
          dims[0] = 2 * N; dims[1] = 256; dims[2] = N / 256; dims[3] = N; dims[4] = 3;
          strides[0] = N * 16; strides[1] = N * 16 * 256; strides[2] = N * N * 16; strides[3] = C / 3;
          box[0] = 2 * W; box[1] = 256; box[2] = N / 256; box[3] = 1; box[4] = 3;
        } else {
          dims[0] = 2 * N; dims[1] = 256; dims[2] = (N / 256) * (N / zb); dims[3] = zb; dims[4] = 3;
          strides[0] = zb * N * 16; strides[1] = 256 * zb * N * 16; strides[2] = N * 16; strides[3] = C / 3;
          box[0] = 2 * W; box[1] = 256; box[2] = N / 256; box[3] = 1; box[4] = 3;
        }
        cuuint32_t es[5] = {1, 1, 1, 1, 1};
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, f, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
          printf("encode failed mode %d zb %d W %d: %d\n", mode, zb, W, (int)r);
          continue;
        }
        const unsigned slot = (unsigned)(W * 3 * n * 16);
        const int nslot = 2;
        const size_t smem = (size_t)slot * nslot;
        const int ntiles = (int)(n / W);
        // a bounded sample: 64 outer lines x all x-tiles
        const int nouter = 64;
        const int nlines = ntiles * nouter;
        cudaFuncSetAttribute(k_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int i = 0; i < 2; ++i) k_tma<2><<<nsm, 256, smem>>>(tm, nlines, ntiles, mode, (int)n, zb, slot, sink);
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        const int reps = 3;
        for (int i = 0; i < reps; ++i) k_tma<2><<<nsm, 256, smem>>>(tm, nlines, ntiles, mode, (int)n, zb, slot, sink);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double moved = (double)nlines * slot;
        const char* names[] = {"z-line ref", "z-line blk", "y-line ref", "y-line blk"};
        printf("%-10s zb=%2d W=%d (box rows %2d B): %8.1f us for %6.2f GB  %7.0f GB/s\n", names[mode], zb, W, 16 * W,
               1e3 * ms / reps, moved / 1e9, moved / (1e6 * ms / reps));
      }
    }
  }
  return 0;
}
