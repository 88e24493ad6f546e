// spmv_inst_nf.cu -- k_spmv<sigma, false, true>: no flagged tiles, heads fit the slots
// (Laplacian-like plans), sigma 1..8
// (one instantiation unit per kernel variant, compiled in parallel).
#include "spmv_kernel.cuh"

namespace csr5g {

SpmvFn spmv_fn_nf(int sigma) {
  switch (sigma) {
    case 1:
      return k_spmv<1, false, true>;
    case 2:
      return k_spmv<2, false, true>;
    case 3:
      return k_spmv<3, false, true>;
    case 4:
      return k_spmv<4, false, true>;
    case 5:
      return k_spmv<5, false, true>;
    case 6:
      return k_spmv<6, false, true>;
    case 7:
      return k_spmv<7, false, true>;
    case 8:
      return k_spmv<8, false, true>;
    default:
      return nullptr;
  }
}

}  // namespace csr5g
