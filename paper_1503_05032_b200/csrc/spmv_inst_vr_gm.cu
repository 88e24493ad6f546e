// spmv_inst_vr_gm.cu -- dispatch over the compile-time gather modes of the VR
// kernel (spmv_inst_vr_gm1..3.cu, spmv_inst_vr_gm5.cu).
#include "spmv_kernel.cuh"

namespace csr5g {

SpmvFn spmv_fn_vr_gm1(int sigma);
SpmvFn spmv_fn_vr_gm2(int sigma);
SpmvFn spmv_fn_vr_gm3(int sigma);
SpmvFn spmv_fn_vr_gm5(int sigma);

SpmvFn spmv_fn_vr_gm(int sigma, int gm) {
  switch (gm) {
    case 1:
      return spmv_fn_vr_gm1(sigma);
    case 2:
      return spmv_fn_vr_gm2(sigma);
    case 3:
      return spmv_fn_vr_gm3(sigma);
    case 5:
      return spmv_fn_vr_gm5(sigma);
    default:
      return nullptr;
  }
}

}  // namespace csr5g
