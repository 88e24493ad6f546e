// spmv_inst_nf2.cu -- k_spmv_nf2<sigma>: NF plans, two tiles per iteration
// (spmv_nf2.cuh), sigma 1..8
// (one instantiation unit per kernel variant, compiled in parallel).
#include "spmv_nf2.cuh"

namespace csr5g {

namespace {
template <int S>
SpmvFn pick_nf2(int sigma) {
  if constexpr (S > kNfMaxSigma) {
    return nullptr;
  } else {
    return sigma == S ? k_spmv_nf2<S> : pick_nf2<S + 1>(sigma);
  }
}
}  // namespace

SpmvFn spmv_fn_nf2(int sigma) { return pick_nf2<1>(sigma); }

}  // namespace csr5g
