// kernel_table.h -- per-length kernel registry shared by the instantiation
// units (inst_<lg>.cu) and the host driver (abi.cu).
#pragma once
#include <cuda_runtime.h>

namespace fftc {

struct KInfo {
  const void* fn = nullptr;
  int threads = 0;     // block size
  int smem = 0;        // dynamic shared memory (bytes)
  int lines = 0;       // lines processed per CTA per loop trip (G)
  int max_active = 0;  // resident CTAs per SM (filled at first use)
  int swz = 0;         // 3-D TMA column passes: tensor maps swizzled over one box row (cols3_lg.cuh)
  int tile_w = 0;      // 3-D TMA column passes: columns per tile (0: col3_tile_w(L))
  int tile_nc = 0;     // ... components per tile (0: 3)
};

// column kernel variants
enum { KC_MID2_BASIC = 0, KC_MID2_EM = 1, KC_MID3_BASIC = 2, KC_MID3_EM = 3, KC_FWD = 4, KC_INV = 5,
       KC_MID2T_BASIC = 6, KC_MID2T_EM = 7,  // *T: TMA tensor-map variants (signature Args, map A, map B)
       KC_MID3T_BASIC = 8, KC_MID3T_EM = 9, KC_FWD3T = 10, KC_INV3T = 11,  // 3-D (Args, Line3, map A, map B, PeerOut*)
       KC_MID3P_BASIC = 12, KC_MID3P_EM = 13, KC_FWD3P = 14,  // the same, outputs to their owning ranks
       KC_COUNT = 15 };
// columns per TMA tile of the 3-D column passes (cols3_lg.cuh: Col3Lg<L>::W)
#ifndef FFTC_COL3_W512
#define FFTC_COL3_W512 4
#endif
// z pass with three components per thread (k_col3_mid); 0: one component per thread
#ifndef FFTC_COL3_MID3
#define FFTC_COL3_MID3 1
#endif
// plain y passes with three components per thread too (k_col3_mid<COL_FWD/COL_INV>)
#ifndef FFTC_COL3_Y3C
#define FFTC_COL3_Y3C 0
#endif
constexpr int col3_tile_w(long long L) { return L <= 256 ? 8 : (L <= 512 ? FFTC_COL3_W512 : 2); }

struct LTable {
  int L = 0;
  int col_w = 0;       // strip width of the column kernels (2-D mid / plain)
  int col3_w = 0;      // strip width of the 3-D mid kernels
  KInfo s1[4];         // sweep 1 per scheme
  KInfo s3[4];         // sweep 3 per scheme
  KInfo s1l[2];        // memory-lean em_sub: sweep 1 of Jq alone, of Rq alone (compact S/T)
  KInfo s3l;           // memory-lean em_sub: sweep 3 over compact S/T
  KInfo col[KC_COUNT];
  KInfo row_fwd, row_inv;  // plain row transforms (operator API)
};

constexpr int MAX_LG = 12;  // supported axis lengths 2 .. 4096

}  // namespace fftc

#define FFTC_DECLARE_FILL(LG) void fftc_fill_table_##LG(fftc::LTable& t);
FFTC_DECLARE_FILL(1)
FFTC_DECLARE_FILL(2)
FFTC_DECLARE_FILL(3)
FFTC_DECLARE_FILL(4)
FFTC_DECLARE_FILL(5)
FFTC_DECLARE_FILL(6)
FFTC_DECLARE_FILL(7)
FFTC_DECLARE_FILL(8)
FFTC_DECLARE_FILL(9)
FFTC_DECLARE_FILL(10)
FFTC_DECLARE_FILL(11)
FFTC_DECLARE_FILL(12)
