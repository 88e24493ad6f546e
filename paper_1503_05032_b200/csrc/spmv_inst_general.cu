// spmv_inst_general.cu -- k_spmv<sigma, false>: the general tile kernel, sigma 1..48 (the
// 64-bit descriptor limit at omega = 32, descriptor.cpp:22-36)
// (one instantiation unit per kernel variant, compiled in parallel).
#include "spmv_kernel.cuh"

namespace csr5g {

SpmvFn spmv_fn_general(int sigma) {
  switch (sigma) {
    case 1:
      return k_spmv<1, false>;
    case 2:
      return k_spmv<2, false>;
    case 3:
      return k_spmv<3, false>;
    case 4:
      return k_spmv<4, false>;
    case 5:
      return k_spmv<5, false>;
    case 6:
      return k_spmv<6, false>;
    case 7:
      return k_spmv<7, false>;
    case 8:
      return k_spmv<8, false>;
    case 9:
      return k_spmv<9, false>;
    case 10:
      return k_spmv<10, false>;
    case 11:
      return k_spmv<11, false>;
    case 12:
      return k_spmv<12, false>;
    case 13:
      return k_spmv<13, false>;
    case 14:
      return k_spmv<14, false>;
    case 15:
      return k_spmv<15, false>;
    case 16:
      return k_spmv<16, false>;
    case 17:
      return k_spmv<17, false>;
    case 18:
      return k_spmv<18, false>;
    case 19:
      return k_spmv<19, false>;
    case 20:
      return k_spmv<20, false>;
    case 21:
      return k_spmv<21, false>;
    case 22:
      return k_spmv<22, false>;
    case 23:
      return k_spmv<23, false>;
    case 24:
      return k_spmv<24, false>;
    case 25:
      return k_spmv<25, false>;
    case 26:
      return k_spmv<26, false>;
    case 27:
      return k_spmv<27, false>;
    case 28:
      return k_spmv<28, false>;
    case 29:
      return k_spmv<29, false>;
    case 30:
      return k_spmv<30, false>;
    case 31:
      return k_spmv<31, false>;
    case 32:
      return k_spmv<32, false>;
    case 33:
      return k_spmv<33, false>;
    case 34:
      return k_spmv<34, false>;
    case 35:
      return k_spmv<35, false>;
    case 36:
      return k_spmv<36, false>;
    case 37:
      return k_spmv<37, false>;
    case 38:
      return k_spmv<38, false>;
    case 39:
      return k_spmv<39, false>;
    case 40:
      return k_spmv<40, false>;
    case 41:
      return k_spmv<41, false>;
    case 42:
      return k_spmv<42, false>;
    case 43:
      return k_spmv<43, false>;
    case 44:
      return k_spmv<44, false>;
    case 45:
      return k_spmv<45, false>;
    case 46:
      return k_spmv<46, false>;
    case 47:
      return k_spmv<47, false>;
    case 48:
      return k_spmv<48, false>;
    default:
      return nullptr;
  }
}

}  // namespace csr5g
