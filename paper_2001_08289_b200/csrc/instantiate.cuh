// instantiate.cuh -- instantiate every sweep kernel for one axis length
// L = 2^FFTC_LG and register it.  Included by the generated inst_<lg>.cu
// files so the ~170 kernels compile in parallel translation units.
#include "sweeps.cuh"
#include "rows_tma.cuh"
#include "cols_tma.cuh"
#include "cols3_tma.cuh"
#include "cols3_lg.cuh"
#include "kernel_table.h"

#ifndef FFTC_TMA_ROWS_MIN
#define FFTC_TMA_ROWS_MIN 512
#endif

#ifndef FFTC_LG
#error "define FFTC_LG before including instantiate.cuh"
#endif

namespace fftc {
namespace inst_detail {

constexpr int L = 1 << FFTC_LG;
// rows: radix-16 lines; sweep 1 splits its channels across thread groups
constexpr int E_ROW = L >= 16 ? 16 : L;
constexpr int T_ROW = L / E_ROW;
constexpr int G_ROW = T_ROW >= 128 ? 1 : 128 / T_ROW;     // sweep 3 / plain: lines per CTA
constexpr int G_ROW1 = T_ROW >= 128 ? 1 : 128 / T_ROW;    // sweep 1, one channel
constexpr int G_ROW2 = T_ROW >= 64 ? 1 : 64 / T_ROW;      // sweep 1, two channels
// columns: radix-8, strips of 2 columns (32-B sectors); 1 column at 4096
#ifndef FFTC_E_COL
#define FFTC_E_COL 8
#endif
constexpr int E_COL = L >= FFTC_E_COL ? FFTC_E_COL : L;
constexpr int T_COL = L / E_COL;
constexpr int W2 = L >= 4096 ? 1 : 2;
constexpr int G2 = (T_COL * W2) >= 64 ? 1 : 64 / (T_COL * W2);
constexpr int W3 = L >= 2048 ? 1 : 2;  // k_col indexes strips assuming W <= 2
constexpr int G3 = (T_COL * W3) >= 64 ? 1 : 64 / (T_COL * W3);
constexpr int WP = 2;  // plain 3-D y passes
constexpr int GP = (T_COL * WP) >= 64 ? 1 : 64 / (T_COL * WP);

template <int C, int W, int G>
constexpr int col_smem() {
  using P = Plan<L, E_COL>;
  constexpr int SKEW = (W > 1) ? 8 / W : 0;
  return G * C * W * (P::LP + SKEW) * (int)sizeof(double2);
}
template <int C, int G>
constexpr int row_smem() {
  return G * C * Plan<L, E_ROW>::LP * (int)sizeof(double2);
}

// component-split 2-D projection sweep (needs at least 8 threads per line
// so that a warp holds whole (t, component, column) quads)
constexpr int E_M2 = L >= 16 ? 16 : L;
constexpr int T_M2 = L / E_M2;
constexpr bool USE_M2 = T_M2 >= 8 && L <= 2048;
constexpr int m2_smem() { return 4 * (Plan<L, E_M2>::LP + 2) * (int)sizeof(double2); }

template <class K>
inline KInfo make(K* fn, int threads, int smem, int lines) {
  KInfo k;
  k.fn = (const void*)fn;
  k.threads = threads;
  k.smem = smem;
  k.lines = lines;
  return k;
}

template <int LL>
inline void fill_tma(LTable& t) {
  if constexpr (LL >= 256 && LL <= 2048) {  // TMA tensor-map 2-D projection sweep
    t.col[KC_MID2T_BASIC] = make(k_mid2_tma<MID_BASIC, LL>, ColTma<LL>::THREADS, ColTma<LL>::SMEM, 1);
    t.col[KC_MID2T_EM] = make(k_mid2_tma<MID_EM, LL>, ColTma<LL>::THREADS, ColTma<LL>::SMEM, 1);
  }
  if constexpr (LL >= 256 && LL <= 1024) {  // TMA tensor-map 3-D column passes
    using K3 = Col3Lg<LL>;
#define FFTC_K3(MODE, PEER) make(k_col3_lg<MODE, LL, PEER>, K3::THREADS, K3::SMEM, 1)
    static_assert(K3::W == col3_tile_w(LL), "host and device tile widths agree");
    t.col[KC_MID3T_BASIC] = FFTC_K3(MID_BASIC, false);
    t.col[KC_MID3T_EM] = FFTC_K3(MID_EM, false);
    t.col[KC_FWD3T] = FFTC_K3(COL_FWD, false);
    t.col[KC_INV3T] = FFTC_K3(COL_INV, false);
    t.col[KC_MID3P_BASIC] = FFTC_K3(MID_BASIC, true);
    t.col[KC_MID3P_EM] = FFTC_K3(MID_EM, true);
    t.col[KC_FWD3P] = FFTC_K3(COL_FWD, true);
#undef FFTC_K3
    for (int kc : {KC_MID3T_BASIC, KC_MID3T_EM, KC_FWD3T, KC_INV3T, KC_MID3P_BASIC, KC_MID3P_EM, KC_FWD3P})
      t.col[kc].swz = K3::W;
    if constexpr (Col3YSel<LL>::Y1) {  // plain y passes on single-component tiles (off by default)
      using KY = typename Col3YSel<LL>::type;
      t.col[KC_FWD3T] = make(k_col3_lg<COL_FWD, LL, false, KY>, KY::THREADS, KY::SMEM, 1);
      t.col[KC_INV3T] = make(k_col3_lg<COL_INV, LL, false, KY>, KY::THREADS, KY::SMEM, 1);
      t.col[KC_FWD3P] = make(k_col3_lg<COL_FWD, LL, true, KY>, KY::THREADS, KY::SMEM, 1);
      for (int kc : {KC_FWD3T, KC_INV3T, KC_FWD3P}) {
        t.col[kc].swz = KY::W;
        t.col[kc].tile_w = KY::W;
        t.col[kc].tile_nc = KY::NC;
      }
    }
#if FFTC_COL3_MID3
    using KM = Col3Mid<LL>;
    t.col[KC_MID3T_BASIC] = make(k_col3_mid<MID_BASIC, LL, false>, KM::THREADS, KM::SMEM, 1);
    t.col[KC_MID3T_EM] = make(k_col3_mid<MID_EM, LL, false>, KM::THREADS, KM::SMEM, 1);
    t.col[KC_MID3P_BASIC] = make(k_col3_mid<MID_BASIC, LL, true>, KM::THREADS, KM::SMEM, 1);
    t.col[KC_MID3P_EM] = make(k_col3_mid<MID_EM, LL, true>, KM::THREADS, KM::SMEM, 1);
    for (int kc : {KC_MID3T_BASIC, KC_MID3T_EM, KC_MID3P_BASIC, KC_MID3P_EM}) t.col[kc].swz = KM::W;
#if FFTC_COL3_Y3C  // plain y passes on the same three-components-per-thread form
    t.col[KC_FWD3T] = make(k_col3_mid<COL_FWD, LL, false>, KM::THREADS, KM::SMEM, 1);
    t.col[KC_INV3T] = make(k_col3_mid<COL_INV, LL, false>, KM::THREADS, KM::SMEM, 1);
    t.col[KC_FWD3P] = make(k_col3_mid<COL_FWD, LL, true>, KM::THREADS, KM::SMEM, 1);
    for (int kc : {KC_FWD3T, KC_INV3T, KC_FWD3P}) t.col[kc].swz = KM::W;
#endif
#endif
  }
  if constexpr (LL >= FFTC_TMA_ROWS_MIN) {  // TMA-staged persistent row sweeps
#define FFTC_TMA(SCH)                                                                                   \
  t.s1[SCH] = make(k_rows_tma<SCH, 1, LL>, RowTma<SCH, 1, LL>::THREADS, RowTma<SCH, 1, LL>::SMEM, 1); \
  t.s3[SCH] = make(k_rows_tma<SCH, 3, LL>, RowTma<SCH, 3, LL>::THREADS, RowTma<SCH, 3, LL>::SMEM, 1);
    FFTC_TMA(BASIC)
    FFTC_TMA(EM)
    FFTC_TMA(BASIC_SUB)
    FFTC_TMA(EM_SUB)
#undef FFTC_TMA
    t.s1l[0] = make(k_rows_tma<EM_SUB, 1, LL, 1>, RowTma<EM_SUB, 1, LL, 1>::THREADS, RowTma<EM_SUB, 1, LL, 1>::SMEM, 1);
    t.s1l[1] = make(k_rows_tma<EM_SUB, 1, LL, 2>, RowTma<EM_SUB, 1, LL, 2>::THREADS, RowTma<EM_SUB, 1, LL, 2>::SMEM, 1);
    t.s3l = make(k_rows_tma<EM_SUB, 3, LL, 3>, RowTma<EM_SUB, 3, LL, 3>::THREADS, RowTma<EM_SUB, 3, LL, 3>::SMEM, 1);
  }
}

}  // namespace inst_detail
}  // namespace fftc

#define FFTC_CAT2(a, b) a##b
#define FFTC_CAT(a, b) FFTC_CAT2(a, b)

void FFTC_CAT(fftc_fill_table_, FFTC_LG)(fftc::LTable& t) {
  using namespace fftc;
  using namespace fftc::inst_detail;
  t.L = L;
  t.col_w = W2;
  t.col3_w = W3;
  const int trow = G_ROW * T_ROW;
  t.s1[BASIC] = make(k_sweep1<BASIC, L, E_ROW, G_ROW1>, G_ROW1 * T_ROW, row_smem<1, G_ROW1>(), G_ROW1);
  t.s1[EM] = make(k_sweep1<EM, L, E_ROW, G_ROW2>, 2 * G_ROW2 * T_ROW, row_smem<2, G_ROW2>(), G_ROW2);
  t.s1[BASIC_SUB] = make(k_sweep1<BASIC_SUB, L, E_ROW, G_ROW1>, G_ROW1 * T_ROW, row_smem<1, G_ROW1>(), G_ROW1);
  t.s1[EM_SUB] = make(k_sweep1<EM_SUB, L, E_ROW, G_ROW2>, 2 * G_ROW2 * T_ROW, row_smem<2, G_ROW2>(), G_ROW2);
  t.s3[BASIC] = make(k_sweep3<BASIC, L, E_ROW, G_ROW>, trow, row_smem<1, G_ROW>(), G_ROW);
  t.s3[EM] = make(k_sweep3<EM, L, E_ROW, G_ROW>, trow, row_smem<1, G_ROW>(), G_ROW);
  t.s3[BASIC_SUB] = make(k_sweep3<BASIC_SUB, L, E_ROW, G_ROW>, trow, row_smem<1, G_ROW>(), G_ROW);
  t.s3[EM_SUB] = make(k_sweep3<EM_SUB, L, E_ROW, G_ROW>, trow, row_smem<1, G_ROW>(), G_ROW);
  fill_tma<L>(t);
  t.row_fwd = make(k_row_plain<false, L, E_ROW, G_ROW>, trow, row_smem<1, G_ROW>(), G_ROW);
  t.row_inv = make(k_row_plain<true, L, E_ROW, G_ROW>, trow, row_smem<1, G_ROW>(), G_ROW);
  if constexpr (USE_M2) {
    t.col[KC_MID2_BASIC] = make(k_mid2<MID_BASIC, L, E_M2>, 4 * T_M2, m2_smem(), 1);
    t.col[KC_MID2_EM] = make(k_mid2<MID_EM, L, E_M2>, 4 * T_M2, m2_smem(), 1);
    t.col_w = 2;
  } else {
    t.col[KC_MID2_BASIC] = make(k_col<MID_BASIC, L, E_COL, W2, 2, G2>, G2 * W2 * T_COL, col_smem<2, W2, G2>(), G2);
    t.col[KC_MID2_EM] = make(k_col<MID_EM, L, E_COL, W2, 2, G2>, G2 * W2 * T_COL, col_smem<2, W2, G2>(), G2);
  }
  t.col[KC_MID3_BASIC] = make(k_col<MID_BASIC, L, E_COL, W3, 3, G3>, G3 * W3 * T_COL, col_smem<3, W3, G3>(), G3);
  t.col[KC_MID3_EM] = make(k_col<MID_EM, L, E_COL, W3, 3, G3>, G3 * W3 * T_COL, col_smem<3, W3, G3>(), G3);
  t.col[KC_FWD] = make(k_col<COL_FWD, L, E_COL, WP, 1, GP>, GP * WP * T_COL, col_smem<1, WP, GP>(), GP);
  t.col[KC_INV] = make(k_col<COL_INV, L, E_COL, WP, 1, GP>, GP * WP * T_COL, col_smem<1, WP, GP>(), GP);
}
