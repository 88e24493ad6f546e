// spmv_inst_vr_gm5.cu -- k_spmv<sigma, true, false, false, 5>: the VR kernel with
// gather mode 5 fixed at compile time (spmv_kernel.cuh, GM), sigma 1..24
// (one instantiation unit per kernel variant, compiled in parallel).
#include "spmv_kernel.cuh"

namespace csr5g {

SpmvFn spmv_fn_vr_gm5(int sigma) { return pick_sigma<1, kVrMaxSigma, true, false, false, 5>(sigma); }

}  // namespace csr5g
