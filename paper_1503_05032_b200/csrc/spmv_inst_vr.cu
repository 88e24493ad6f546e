// spmv_inst_vr.cu -- k_spmv<sigma, true>: values loaded with the gathers (random-gather
// plans), sigma 1..24
// (one instantiation unit per kernel variant, compiled in parallel).
#include "spmv_kernel.cuh"

namespace csr5g {

SpmvFn spmv_fn_vr(int sigma) {
  switch (sigma) {
    case 1:
      return k_spmv<1, true>;
    case 2:
      return k_spmv<2, true>;
    case 3:
      return k_spmv<3, true>;
    case 4:
      return k_spmv<4, true>;
    case 5:
      return k_spmv<5, true>;
    case 6:
      return k_spmv<6, true>;
    case 7:
      return k_spmv<7, true>;
    case 8:
      return k_spmv<8, true>;
    case 9:
      return k_spmv<9, true>;
    case 10:
      return k_spmv<10, true>;
    case 11:
      return k_spmv<11, true>;
    case 12:
      return k_spmv<12, true>;
    case 13:
      return k_spmv<13, true>;
    case 14:
      return k_spmv<14, true>;
    case 15:
      return k_spmv<15, true>;
    case 16:
      return k_spmv<16, true>;
    case 17:
      return k_spmv<17, true>;
    case 18:
      return k_spmv<18, true>;
    case 19:
      return k_spmv<19, true>;
    case 20:
      return k_spmv<20, true>;
    case 21:
      return k_spmv<21, true>;
    case 22:
      return k_spmv<22, true>;
    case 23:
      return k_spmv<23, true>;
    case 24:
      return k_spmv<24, true>;
    default:
      return nullptr;
  }
}

}  // namespace csr5g
