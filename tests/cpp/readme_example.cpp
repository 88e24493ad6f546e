// The reference README's library example (proj/README.md:115-123), compiled
// unchanged against the csr5:: drop-in and linked through find_package(csr5)
// (tests/cpp/CMakeLists.txt).  Prints "README OK" when y matches the
// reference kernel within 1e-12.
#include <csr5/format.hpp>
#include <csr5/matrix_market.hpp>
#include <csr5/spmv.hpp>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>

int main() {
  {
    std::ofstream f("matrix.mtx");
    f << "%%MatrixMarket matrix coordinate real general\n5 5 9\n1 1 4\n1 2 -1\n2 2 4\n"
         "3 1 -1\n3 3 4\n4 4 4\n4 5 -1\n5 3 -1\n5 5 4\n";
  }
  csr5::DenseVector x{1.0, 2.0, 3.0, 4.0, 5.0};
  // ---- README.md:119-121, verbatim ----
  csr5::CsrMatrix a = csr5::load_matrix_market("matrix.mtx");
  csr5::Csr5Matrix a5 = csr5::csr_to_csr5(a, csr5::TuningParams{});
  csr5::DenseVector y = csr5::spmv_csr5(a5, x);
  // ----
  const csr5::DenseVector ref = csr5::dense_spmv_oracle(a, x);
  double err = 0.0;
  for (std::size_t i = 0; i < y.size(); ++i)
    err = std::max(err, std::abs(y[i] - ref[i]) / std::max(1.0, std::abs(ref[i])));
  if (a.nnz() != 9 || y.size() != 5 || err > 1e-12) {
    std::printf("README FAILED: nnz=%lld err=%g\n", (long long)a.nnz(), err);
    return 1;
  }
  std::printf("README OK (omega=%lld sigma=%lld)\n", (long long)a5.omega(), (long long)a5.sigma());
  return 0;
}
