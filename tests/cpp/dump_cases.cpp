// csr5::dump_format over the C++ drop-in for matrices given as files (one per
// argument: "m n sigma", then row_ptr, col_idx and the values as hex floats);
// writes <file>.dump.  tests/test_gpu_dump.py compares every output byte for
// byte with the reference's own dump_format (tests/golden/ref_dumps.json.gz).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <string>

#include "csr5/format.hpp"

int main(int argc, char** argv) {
  for (int k = 1; k < argc; ++k) {
    std::ifstream in(argv[k]);
    csr5::CsrMatrix a;
    csr5::index_t sigma = 0;
    in >> a.m >> a.n >> sigma;
    a.row_ptr.resize(static_cast<std::size_t>(a.m) + 1);
    for (auto& v : a.row_ptr) in >> v;
    a.col_idx.resize(static_cast<std::size_t>(a.nnz()));
    for (auto& v : a.col_idx) in >> v;
    a.val.resize(static_cast<std::size_t>(a.nnz()));
    std::string tok;
    for (auto& v : a.val) {
      in >> tok;
      v = std::strtod(tok.c_str(), nullptr);
    }
    if (!in) {
      std::cerr << "bad input " << argv[k] << "\n";
      return 2;
    }
    const csr5::Csr5Matrix a5 = csr5::csr_to_csr5(a, csr5::TuningParams{.omega = 32, .sigma = sigma});
    std::ofstream out(std::string(argv[k]) + ".dump");
    csr5::dump_format(a5, out);
  }
  std::printf("DUMPS OK %d\n", argc - 1);
  return 0;
}
