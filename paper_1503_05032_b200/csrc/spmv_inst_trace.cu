// spmv_inst_trace.cu -- k_spmv<sigma, false, false, true>: one tile's contributions
// (csr5g_spmv_tile, the spmv_csr5_tile test hook), sigma 1..48
// (one instantiation unit per kernel variant, compiled in parallel).
#include "spmv_kernel.cuh"

namespace csr5g {

SpmvFn spmv_fn_trace(int sigma) {
  switch (sigma) {
    case 1:
      return k_spmv<1, false, false, true>;
    case 2:
      return k_spmv<2, false, false, true>;
    case 3:
      return k_spmv<3, false, false, true>;
    case 4:
      return k_spmv<4, false, false, true>;
    case 5:
      return k_spmv<5, false, false, true>;
    case 6:
      return k_spmv<6, false, false, true>;
    case 7:
      return k_spmv<7, false, false, true>;
    case 8:
      return k_spmv<8, false, false, true>;
    case 9:
      return k_spmv<9, false, false, true>;
    case 10:
      return k_spmv<10, false, false, true>;
    case 11:
      return k_spmv<11, false, false, true>;
    case 12:
      return k_spmv<12, false, false, true>;
    case 13:
      return k_spmv<13, false, false, true>;
    case 14:
      return k_spmv<14, false, false, true>;
    case 15:
      return k_spmv<15, false, false, true>;
    case 16:
      return k_spmv<16, false, false, true>;
    case 17:
      return k_spmv<17, false, false, true>;
    case 18:
      return k_spmv<18, false, false, true>;
    case 19:
      return k_spmv<19, false, false, true>;
    case 20:
      return k_spmv<20, false, false, true>;
    case 21:
      return k_spmv<21, false, false, true>;
    case 22:
      return k_spmv<22, false, false, true>;
    case 23:
      return k_spmv<23, false, false, true>;
    case 24:
      return k_spmv<24, false, false, true>;
    case 25:
      return k_spmv<25, false, false, true>;
    case 26:
      return k_spmv<26, false, false, true>;
    case 27:
      return k_spmv<27, false, false, true>;
    case 28:
      return k_spmv<28, false, false, true>;
    case 29:
      return k_spmv<29, false, false, true>;
    case 30:
      return k_spmv<30, false, false, true>;
    case 31:
      return k_spmv<31, false, false, true>;
    case 32:
      return k_spmv<32, false, false, true>;
    case 33:
      return k_spmv<33, false, false, true>;
    case 34:
      return k_spmv<34, false, false, true>;
    case 35:
      return k_spmv<35, false, false, true>;
    case 36:
      return k_spmv<36, false, false, true>;
    case 37:
      return k_spmv<37, false, false, true>;
    case 38:
      return k_spmv<38, false, false, true>;
    case 39:
      return k_spmv<39, false, false, true>;
    case 40:
      return k_spmv<40, false, false, true>;
    case 41:
      return k_spmv<41, false, false, true>;
    case 42:
      return k_spmv<42, false, false, true>;
    case 43:
      return k_spmv<43, false, false, true>;
    case 44:
      return k_spmv<44, false, false, true>;
    case 45:
      return k_spmv<45, false, false, true>;
    case 46:
      return k_spmv<46, false, false, true>;
    case 47:
      return k_spmv<47, false, false, true>;
    case 48:
      return k_spmv<48, false, false, true>;
    default:
      return nullptr;
  }
}

}  // namespace csr5g
