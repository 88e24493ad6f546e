// spmv_inst_gm4.cu -- k_spmv<sigma, false, NF, false, 4>: the general (sigma 1..48)
// and NF (sigma 1..8) kernels with plain read-only x loads fixed at compile
// time (local plans, x_mode 4; spmv_kernel.cuh, GM)
// (one instantiation unit per kernel variant, compiled in parallel).
#include "spmv_kernel.cuh"

namespace csr5g {

SpmvFn spmv_fn_local_gm4(int sigma, bool nf) {
  return nf ? pick_sigma<1, kNfMaxSigma, false, true, false, 4>(sigma)
            : pick_sigma<1, 48, false, false, false, 4>(sigma);
}

}  // namespace csr5g
