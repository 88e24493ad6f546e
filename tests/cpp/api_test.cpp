// Exercises the csr5:: drop-in (include/csr5/*.hpp) on the GPU beyond the
// reference's own cases (tests/cpp/ref_cases.cpp): sigma auto, both modes,
// the reference's error texts, the pipelined host batch (csr5/gpu.hpp),
// concurrent calls from host threads, Matrix Market ingest.  Built through
// find_package(csr5); run by tests/test_gpu_cpp.py; prints "API OK".
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "csr5/format.hpp"
#include "csr5/gpu.hpp"
#include "csr5/matrix_market.hpp"
#include "csr5/spmv.hpp"

using namespace csr5;

static int failures = 0;
#define CHECK(c)                                                     \
  do {                                                               \
    if (!(c)) {                                                      \
      std::printf("CHECK failed: %s (line %d)\n", #c, __LINE__);     \
      ++failures;                                                    \
    }                                                                \
  } while (0)

// sequential row-order oracle (the reference's dense_spmv_oracle, csr.cpp:85-98)
static DenseVector oracle(const CsrMatrix& a, const DenseVector& x) {
  DenseVector y((std::size_t)a.m, 0.0);
  for (index_t i = 0; i < a.m; ++i) {
    double s = 0.0;
    for (index_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) s += a.val[k] * x[a.col_idx[k]];
    y[i] = s;
  }
  return y;
}

static double max_rel(const DenseVector& y, const DenseVector& r) {
  double w = 0.0;
  for (std::size_t i = 0; i < y.size(); ++i)
    w = std::max(w, std::abs(y[i] - r[i]) / std::max(1.0, std::abs(r[i])));
  return w;
}

static CsrMatrix random_csr(unsigned long long seed, index_t m, index_t n, double density) {
  CsrMatrix a;
  a.m = m;
  a.n = n;
  a.row_ptr.push_back(0);
  unsigned long long s = seed;
  auto next = [&] {
    s = s * 6364136223846793005ULL + 1442695040888963407ULL;
    return s >> 11;
  };
  for (index_t i = 0; i < m; ++i) {
    for (index_t j = 0; j < n; ++j)
      if ((next() % 1000000) < density * 1e6) {
        a.col_idx.push_back(j);
        a.val.push_back(0.5 + (double)(next() % 1000000) * 1e-6);
      }
    a.row_ptr.push_back((index_t)a.col_idx.size());
  }
  return a;
}

int main() {
  // 8x8 with 34 nonzeros (test_format.cpp:30-44)
  {
    const std::vector<std::vector<index_t>> cols = {{0, 1, 2, 3, 4, 5}, {}, {0, 2, 4, 6, 7},
                                                    {1, 3, 5, 6, 7}, {0, 1, 2, 3, 4, 5, 6},
                                                    {1, 2, 3, 5, 6, 7}, {0, 3, 6}, {2, 5}};
    CsrMatrix a;
    a.m = a.n = 8;
    a.row_ptr.push_back(0);
    double v = 1.0;
    for (auto& r : cols) {
      for (index_t c : r) {
        a.col_idx.push_back(c);
        a.val.push_back(v++);
      }
      a.row_ptr.push_back((index_t)a.col_idx.size());
    }
    Csr5Matrix a5 = csr_to_csr5(a, TuningParams{.sigma = 1});  // B = 32: 1 tile + tail 2
    CHECK(a5.p == 2 && a5.p_complete == 1 && a5.tail_len == 2);
    const DenseVector x(8, 1.0);
    CHECK(max_rel(spmv_csr5(a5, x), oracle(a, x)) <= 1e-12);
    CHECK(csr5_to_csr(a5) == a);
    std::ostringstream out;
    dump_format(a5, out);
    CHECK(out.str().find("tile 0:") != std::string::npos);
    CHECK(out.str().find("tail nnz=2") != std::string::npos);
  }
  // random matrices over sigma, both modes
  for (index_t sigma : {1, 4, 16, 17, 18, 27, 48}) {
    const CsrMatrix a = random_csr(1000 + sigma, 700, 500, 0.03);
    DenseVector x((std::size_t)a.n);
    for (std::size_t i = 0; i < x.size(); ++i) x[i] = 0.5 + 0.001 * (double)(i % 997);
    Csr5Matrix a5 = csr_to_csr5(a, TuningParams{.sigma = sigma});
    const DenseVector ref = oracle(a, x);
    CHECK(max_rel(spmv_csr5(a5, x), ref) <= 1e-12);
    CHECK(max_rel(spmv_csr5(a5, x, SpmvMode::atomic), ref) <= 1e-12);
    CHECK(csr5_to_csr(a5) == a);
    CHECK(a5.sigma() == sigma);
  }
  // reference error behaviour
  {
    const CsrMatrix a = random_csr(7, 20, 30, 0.2);
    bool threw = false;
    try {
      (void)csr_to_csr5(a, TuningParams{.omega = 4, .sigma = 16});
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
    threw = false;
    try {
      (void)csr_to_csr5(a, TuningParams{.omega = 32, .sigma = 60});
    } catch (const std::invalid_argument& e) {
      threw = std::string(e.what()).find("smaller sigma") != std::string::npos;
    }
    CHECK(threw);
    Csr5Matrix a5 = csr_to_csr5(a, TuningParams{});
    threw = false;
    try {
      (void)spmv_csr5(a5, DenseVector(29, 1.0));
    } catch (const std::invalid_argument& e) {
      threw = std::string(e.what()) == "spmv: x has length 29, expected 30";
    }
    CHECK(threw);
  }
  // batch of host vectors through the pipelined entry point
  {
    const CsrMatrix a = random_csr(99, 900, 800, 0.02);
    Csr5Matrix a5 = csr_to_csr5(a, TuningParams{});
    std::vector<DenseVector> xs(5, DenseVector((std::size_t)a.n)), ys(5);
    std::vector<const double*> px;
    std::vector<double*> py;
    for (std::size_t k = 0; k < xs.size(); ++k) {
      for (std::size_t i = 0; i < xs[k].size(); ++i) xs[k][i] = 0.25 + 0.01 * (double)((i + k) % 89);
      ys[k].assign((std::size_t)a.m, -1.0);
      px.push_back(xs[k].data());
      py.push_back(ys[k].data());
    }
    spmv_csr5_batch(a5, px, py);
    for (std::size_t k = 0; k < xs.size(); ++k) CHECK(ys[k] == spmv_csr5(a5, xs[k]));
  }
  // one matrix, spmv_csr5 from several host threads at once (the reference's
  // types are shareable read-only): every result equals the
  // single-threaded one bit for bit (deterministic mode)
  {
    const CsrMatrix a = random_csr(77, 900, 700, 0.05);
    const Csr5Matrix a5 = csr_to_csr5(a, TuningParams{});
    const Csr5Matrix copy = a5;  // value semantics: copies share one device handle
    const int T = 6;
    std::vector<DenseVector> xs(T, DenseVector((std::size_t)a.n)), ref(T), got(T);
    for (int t = 0; t < T; ++t) {
      for (std::size_t i = 0; i < xs[t].size(); ++i) xs[t][i] = 0.5 + 0.003 * (double)((7 * i + t) % 331);
      ref[t] = spmv_csr5(a5, xs[t]);
    }
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        for (int r = 0; r < 20; ++r) got[t] = spmv_csr5(t % 2 ? copy : a5, xs[t]);
      });
    for (auto& x : th) x.join();
    for (int t = 0; t < T; ++t) CHECK(got[t] == ref[t]);
  }
  // Matrix Market -> coo_to_csr on the device -> CSR5
  {
    const char* path = "api_test.mtx";
    {
      std::ofstream f(path);
      f << "%%MatrixMarket matrix coordinate real symmetric\n% c\n4 4 5\n1 1 2.0\n2 1 -1\n"
           "3 3 4.5\n4 2 1e-3\n2 1 0.5\n";
    }
    const CsrMatrix a = load_matrix_market(path);
    CHECK(a.m == 4 && a.n == 4 && a.nnz() == 6);
    CHECK((a.row_ptr == std::vector<index_t>{0, 2, 4, 5, 6}));
    CHECK((a.col_idx == std::vector<index_t>{0, 1, 0, 3, 2, 1}));
    CHECK((a.val == std::vector<double>{2.0, -0.5, -0.5, 1e-3, 4.5, 1e-3}));
    const DenseVector x{1.0, 2.0, 3.0, 4.0};
    CHECK(max_rel(spmv_csr5(csr_to_csr5(a, TuningParams{}), x), oracle(a, x)) <= 1e-12);
    std::istringstream text("%%MatrixMarket matrix coordinate pattern general\n2 3 2\n1 3\n2 1\n");
    const MatrixMarketData d = read_matrix_market(text);
    CHECK(d.m == 2 && d.n == 3 && d.entries.size() == 2 && d.entries[0].col == 2 &&
          d.entries[1].value == 1.0);
    bool threw = false;
    try {
      (void)coo_to_csr({{0, 0, 1.0}, {2, 5, 1.0}}, 3, 3);
    } catch (const std::invalid_argument& e) {
      threw = std::string(e.what()) == "coo entry 1 out of bounds: (2, 5) for a 3x3 matrix";
    }
    CHECK(threw);
    threw = false;
    try {
      (void)read_matrix_market("does_not_exist.mtx");
    } catch (const std::runtime_error& e) {
      threw = std::string(e.what()) == "matrix market: cannot open 'does_not_exist.mtx'";
    }
    CHECK(threw);
  }
  if (failures) {
    std::printf("API FAILED (%d)\n", failures);
    return 1;
  }
  std::printf("API OK\n");
  return 0;
}
