// csr5/matrix_market.hpp -- drop-in for the reference's matrix_market.hpp
// (matrix_market.cpp:38-103): the library's parser (ingest.cu) with the
// reference's accepted headers, 0-based indices, symmetric expansion and
// std::runtime_error texts.
#pragma once

#include <istream>
#include <iterator>
#include <string>
#include <vector>

#include "csr5/csr.hpp"

namespace csr5 {

struct MatrixMarketData {
  std::vector<CooEntry> entries;
  index_t m = 0;
  index_t n = 0;
};

namespace detail {
inline MatrixMarketData take_coo(csr5g_coo h, std::int64_t m, std::int64_t n, std::int64_t k) {
  std::vector<index_t> r((std::size_t)k), c((std::size_t)k);
  std::vector<double> v((std::size_t)k);
  const int rc = csr5g_coo_get(h, r.data(), c.data(), v.data());
  csr5g_coo_release(h);
  check(rc);
  MatrixMarketData d;
  d.m = m;
  d.n = n;
  d.entries.reserve((std::size_t)k);
  for (std::size_t q = 0; q < (std::size_t)k; ++q) d.entries.push_back({r[q], c[q], v[q]});
  return d;
}
}  // namespace detail

inline MatrixMarketData read_matrix_market(std::istream& in) {
  const std::string text{std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()};
  csr5g_coo h = nullptr;
  std::int64_t m = 0, n = 0, k = 0;
  detail::check(csr5g_mm_parse(text.data(), static_cast<std::int64_t>(text.size()), &h, &m, &n, &k));
  return detail::take_coo(h, m, n, k);
}

inline MatrixMarketData read_matrix_market(const std::string& path) {
  csr5g_coo h = nullptr;
  std::int64_t m = 0, n = 0, k = 0;
  detail::check(csr5g_mm_read(path.c_str(), &h, &m, &n, &k));
  return detail::take_coo(h, m, n, k);
}

/// read_matrix_market followed by coo_to_csr (on the current CUDA device).
inline CsrMatrix load_matrix_market(const std::string& path) {
  MatrixMarketData d = read_matrix_market(path);
  return coo_to_csr(std::move(d.entries), d.m, d.n);
}

}  // namespace csr5
