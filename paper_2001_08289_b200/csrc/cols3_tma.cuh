// cols3_tma.cuh -- TMA helpers of the 3-D column passes (cols3_lg.cuh): tile
// load / store / bulk-copy PTX wrappers and the tensor-map coordinates of a
// tile.  (Round 1's kernel k_col3_tma, one component of one column per thread
// with the column's threads spread over eight warps and CTA-wide barriers,
// lived here; cols3_lg.cuh replaced it -- see DESIGN.md section 3.  Its last
// round-2 form, with barriers removed around the projection, failed the
// 1024-line parity fixture c4first and is gone; git history keeps it.)
#pragma once
#include "cols_tma.cuh"
#include "kernel_table.h"

namespace fftc {

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

}  // namespace fftc
