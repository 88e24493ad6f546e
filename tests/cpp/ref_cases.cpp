// omega = 32 variants of the reference's own test cases
// (proj/tests/test_format.cpp, test_spmv.cpp, test_descriptor.cpp,
// test_tuning.cpp), written against the csr5:: drop-in headers exactly as the
// originals are written against proj/core/include/csr5 -- same includes,
// same calls, same checks -- with the tile width the GPU requires (one warp
// lane per tile column) and the expected numbers that follow from it.
// Built through find_package(csr5) (tests/cpp/CMakeLists.txt); run on the GPU
// by tests/test_gpu_cpp.py.
#include "mini_doctest.h"

#include <bit>
#include <cstring>
#include <map>
#include <random>
#include <sstream>
#include <stdexcept>
#include <thread>

#include "csr5/format.hpp"
#include "csr5/spmv.hpp"
#include "csr5/tuning.hpp"

using namespace csr5;

namespace {

// random canonical matrix through COO entries (duplicates summed) and a
// random positive x -- the reference's test_helpers.hpp conventions
CsrMatrix random_csr(std::mt19937_64& rng, index_t m, index_t n, index_t nnz_target) {
  std::vector<CooEntry> e;
  for (index_t k = 0; k < nnz_target; ++k) {
    const index_t r = static_cast<index_t>(rng() % static_cast<std::uint64_t>(m));
    const index_t c = static_cast<index_t>(rng() % static_cast<std::uint64_t>(n));
    e.push_back({r, c, 0.5 + static_cast<double>(rng() >> 11) * 0x1.0p-53});
  }
  return coo_to_csr(std::move(e), m, n);
}
DenseVector random_x(std::mt19937_64& rng, index_t n) {
  DenseVector x(static_cast<std::size_t>(n));
  for (double& v : x) v = 0.5 + static_cast<double>(rng() >> 11) * 0x1.0p-53;
  return x;
}
double max_relative_error(const DenseVector& y, const DenseVector& ref) {
  double w = 0.0;
  for (std::size_t i = 0; i < y.size(); ++i)
    w = std::max(w, std::abs(y[i] - ref[i]) / std::max(1.0, std::abs(ref[i])));
  return w;
}
void check_close(const DenseVector& y, const DenseVector& ref, double tol = 1e-12) {
  REQUIRE(y.size() == ref.size());
  CHECK(max_relative_error(y, ref) <= tol);
}

// 8x8 with 34 nonzeros; row lengths 6,0,5,5,7,6,3,2 (test_format.cpp:30-44)
CsrMatrix eight_by_eight() {
  std::vector<CooEntry> entries;
  const std::vector<std::vector<index_t>> cols = {
      {0, 1, 2, 3, 4, 5}, {}, {0, 2, 4, 6, 7}, {1, 3, 5, 6, 7},
      {0, 1, 2, 3, 4, 5, 6}, {1, 2, 3, 5, 6, 7}, {0, 3, 6}, {2, 5}};
  double v = 1.0;
  for (index_t r = 0; r < 8; ++r)
    for (index_t c : cols[static_cast<std::size_t>(r)]) entries.push_back({r, c, v++});
  CsrMatrix a = coo_to_csr(std::move(entries), 8, 8);
  REQUIRE(a.nnz() == 34);
  REQUIRE(a.row_ptr[4] == 16);
  return a;
}

CsrMatrix dense_block(index_t m, index_t n) {  // every entry present
  std::vector<CooEntry> e;
  for (index_t r = 0; r < m; ++r)
    for (index_t c = 0; c < n; ++c) e.push_back({r, c, 1.0 + static_cast<double>((r * n + c) % 7)});
  return coo_to_csr(std::move(e), m, n);
}

}  // namespace

// ---------------------------------------------------------------- tuning ----
TEST_CASE("sigma selection table") {  // test_tuning.cpp:16-25
  const TuningParams b{.r = 2, .s = 10, .t = 100, .u = 4};
  CHECK(select_sigma(1.0, b) == 2);
  CHECK(select_sigma(7.4, b) == 7);
  CHECK(select_sigma(50.0, b) == 10);
  CHECK(select_sigma(1000.0, b) == 4);
  CHECK(select_sigma(3.0, b, 9) == 9);
  const TuningParams d{};
  CHECK(select_sigma(4.0, d) == 4);
  CHECK(select_sigma(32.0, d) == 32);
  CHECK(select_sigma(256.0, d) == 32);
  CHECK(select_omega() == 32);
  CHECK(select_omega(8) == 8);
  CHECK_THROWS_AS((TuningParams{.omega = 1, .sigma = 1}.validate()), std::invalid_argument);
  CHECK_THROWS_AS((TuningParams{.r = 5, .s = 4}.validate()), std::invalid_argument);
}

// ------------------------------------------------------------ descriptor ----
TEST_CASE("descriptor layout and packing at omega = 32") {  // test_descriptor.cpp:26-98
  const DescriptorLayout l16 = make_descriptor_layout(32, 16);
  CHECK(l16.y_offset_bits == 9);
  CHECK(l16.seg_offset_bits == 5);
  CHECK(l16.column_bits() == 30);
  CHECK(l16.word_bits == 32);
  CHECK(make_descriptor_layout(32, 27).word_bits == 64);
  CHECK_THROWS_AS(make_descriptor_layout(32, 60), std::invalid_argument);
  std::mt19937_64 rng(5);
  for (index_t sigma : {1, 5, 16, 17, 18, 27, 48}) {
    const DescriptorLayout l = make_descriptor_layout(32, sigma);
    TileDescriptor d;
    for (int i = 0; i < 32; ++i) {
      d.y_offset.push_back(static_cast<index_t>(rng() % static_cast<std::uint64_t>(32 * sigma)));
      d.seg_offset.push_back(static_cast<index_t>(rng() % 32));
      for (index_t j = 0; j < sigma; ++j) d.bit_flag.push_back(static_cast<std::uint8_t>(rng() & 1));
    }
    const auto w = pack_tile_descriptor(d, l);
    CHECK(unpack_tile_descriptor(w, l) == d);
  }
}

// ---------------------------------------------------------------- format ----
TEST_CASE("flagged first tile stores negative zero") {  // test_format.cpp:70-76
  CHECK(encode_tile_ptr(0, true, 32) == 0x80000000ull);
  CHECK(encode_tile_ptr(5, true, 64) == 0x8000000000000005ull);
  CHECK(decode_tile_ptr_row(0x80000000ull, 32) == 0);
  CHECK(decode_tile_ptr_flag(0x80000000ull, 32));
  CHECK(tile_ptr_bits_for_rows(index_t{1} << 31) == 64);
  const std::vector<index_t> rp{0, 2, 2, 5, 8};
  CHECK(row_of_nonzero(rp, 1) == 0);
  CHECK(row_of_nonzero(rp, 2) == 2);
  CHECK(row_of_nonzero(rp, 8) == 3);
}

TEST_CASE("conversion splits an 8x8/34 matrix into 1 complete tile + tail of 2") {
  const CsrMatrix a = eight_by_eight();
  const Csr5Matrix a5 = csr_to_csr5(a, TuningParams{.omega = 32, .sigma = 1});
  CHECK(a5.p == 2);
  CHECK(a5.p_complete == 1);
  CHECK(a5.tail_len == 2);
  CHECK(a5.tile_row(1) == 7);  // nonzero 32 sits in row 7
  CHECK(a5.tile_row(2) == 7);  // closing entry: m - 1
  CHECK(a5.tile_has_empty_rows(0));
  CHECK_FALSE(a5.tile_has_empty_rows(1));
  CHECK(a5.row_ptr == a.row_ptr);
  CHECK(a5.metadata_bytes() == 3 * 4 + 32 * 4);
}

TEST_CASE("conversion of the empty matrix") {  // test_format.cpp:175-183
  const CsrMatrix a = coo_to_csr({}, 5, 5);
  const Csr5Matrix a5 = csr_to_csr5(a, TuningParams{});
  CHECK(a5.p == 0);
  CHECK(a5.p_complete == 0);
  CHECK(a5.tile_desc.size() == 0);
  CHECK(a5.col_idx.empty());
  CHECK(csr5_to_csr(a5) == a);
}

TEST_CASE("round-trip is bit-exact across tile shapes") {  // test_format.cpp:185-204
  std::mt19937_64 rng(23);
  for (index_t sigma : {1, 2, 4, 12, 16, 27, 48}) {
    for (int trial = 0; trial < 8; ++trial) {
      const index_t m = 1 + static_cast<index_t>(rng() % 80);
      const index_t n = 1 + static_cast<index_t>(rng() % 80);
      const index_t nnz = static_cast<index_t>(rng() % static_cast<std::uint64_t>(m * n + 1));
      const CsrMatrix a = random_csr(rng, m, n, nnz);
      TuningParams params{};
      params.sigma = sigma;
      const Csr5Matrix a5 = csr_to_csr5(a, params);
      CHECK(csr5_to_csr(a5) == a);
    }
  }
}

TEST_CASE("round-trip when nnz is an exact tile multiple") {  // test_format.cpp:206-214
  const CsrMatrix a = dense_block(16, 16);
  const Csr5Matrix a5 = csr_to_csr5(a, TuningParams{.omega = 32, .sigma = 4});
  CHECK(a5.p == 2);
  CHECK(a5.p_complete == 2);
  CHECK(a5.tail_len == 0);
  CHECK(a5.tile_row(2) == 15);  // closing entry decodes to the final row
  CHECK(csr5_to_csr(a5) == a);
}

TEST_CASE("parallel and sequential conversion produce identical matrices") {
  std::mt19937_64 rng(29);
  const CsrMatrix a = random_csr(rng, 120, 90, 2500);
  const TuningParams params{.omega = 32, .sigma = 12};
  const Csr5Matrix par = csr_to_csr5(a, params, /*parallel=*/true);
  const Csr5Matrix seq = csr_to_csr5(a, params, /*parallel=*/false);
  CHECK(par.tile_ptr == seq.tile_ptr);
  CHECK(par.tile_desc == seq.tile_desc);
  CHECK(par.empty_offset == seq.empty_offset);
  CHECK(par.col_idx == seq.col_idx);
  CHECK(par.val == seq.val);
}

TEST_CASE("conversion rejects an invalid tile shape") {  // test_format.cpp:229-232
  const CsrMatrix a = coo_to_csr({{0, 0, 1.0}}, 1, 1);
  CHECK_THROWS_AS(csr_to_csr5(a, TuningParams{.omega = 1, .sigma = 1}), std::invalid_argument);
  CHECK_THROWS_AS(csr_to_csr5(a, TuningParams{.omega = 4, .sigma = 16}), std::invalid_argument);
  CHECK_THROWS_AS(csr_to_csr5(a, TuningParams{.omega = 32, .sigma = 60}), std::invalid_argument);
}

TEST_CASE("format invariants hold on random matrices") {  // test_format.cpp:234-313
  std::mt19937_64 rng(31);
  for (int trial = 0; trial < 40; ++trial) {
    const index_t m = 1 + static_cast<index_t>(rng() % 200);
    const index_t n = 1 + static_cast<index_t>(rng() % 200);
    const CsrMatrix a = random_csr(rng, m, n, static_cast<index_t>(rng() % 2400));
    const TuningParams params{.omega = 32, .sigma = 4};
    const Csr5Matrix a5 = csr_to_csr5(a, params);

    index_t prev_row = 0;
    for (index_t tid = 0; tid <= a5.p; ++tid) {
      CHECK(a5.tile_row(tid) >= prev_row);
      prev_row = a5.tile_row(tid);
      if (a5.m > 0) CHECK(a5.tile_row(tid) < a5.m);
    }
    for (index_t tid = 0; tid < a5.p_complete; ++tid) {
      const TileDescriptor d = a5.descriptor(tid);
      CHECK(d.bit_flag[0] == 1);
      index_t heads_before = 0, total_heads = 0;
      for (index_t i = 0; i < params.omega; ++i) {
        CHECK(d.y_offset[static_cast<std::size_t>(i)] == heads_before);
        index_t col_heads = 0;
        for (index_t j = 0; j < params.sigma; ++j)
          col_heads += d.bit_flag[static_cast<std::size_t>(i * params.sigma + j)];
        heads_before += col_heads;
        total_heads += col_heads;
        const index_t seg = d.seg_offset[static_cast<std::size_t>(i)];
        CHECK(seg >= 0);
        CHECK(seg <= params.omega - 1 - i);
      }
      // the y_offset / seg_offset rule of the reference, from the bit flags
      const auto [yo, so] = generate_y_and_seg_offset(d.bit_flag, params.omega, params.sigma);
      CHECK(yo == d.y_offset);
      CHECK(so == d.seg_offset);
      if (a5.tile_has_empty_rows(tid)) {
        const index_t begin = a5.empty_offset_ptr[static_cast<std::size_t>(tid)];
        const index_t end = a5.empty_offset_ptr[static_cast<std::size_t>(tid + 1)];
        CHECK(end - begin == total_heads);
        index_t k = begin;
        for (index_t i = 0; i < params.omega; ++i)
          for (index_t j = 0; j < params.sigma; ++j) {
            if (!d.bit_flag[static_cast<std::size_t>(i * params.sigma + j)]) continue;
            const index_t g = tile_logical_index(tid, params.omega, params.sigma, i, j);
            const index_t row = a5.tile_row(tid) + a5.empty_offset[static_cast<std::size_t>(k)];
            CHECK(a5.row_ptr[static_cast<std::size_t>(row)] <= g);
            CHECK(g < a5.row_ptr[static_cast<std::size_t>(row + 1)]);
            ++k;
          }
        const auto eo = generate_empty_offset(a, tid, a5.tile_row(tid), d.bit_flag, params.omega,
                                              params.sigma);
        CHECK(std::equal(eo.begin(), eo.end(), a5.empty_offset.begin() + begin));
      } else {
        CHECK(a5.empty_offset_ptr[static_cast<std::size_t>(tid)] ==
              a5.empty_offset_ptr[static_cast<std::size_t>(tid + 1)]);
      }
    }
  }
}

TEST_CASE("dump_format lists one tile per line") {  // test_format.cpp:315-326
  const CsrMatrix a = eight_by_eight();
  const Csr5Matrix a5 = csr_to_csr5(a, TuningParams{.omega = 32, .sigma = 1});
  std::ostringstream out;
  dump_format(a5, out);
  const std::string text = out.str();
  CHECK(text.find("tile 0:") != std::string::npos);
  CHECK(text.find("tile 1:") != std::string::npos);
  CHECK(text.find("tail") != std::string::npos);
  CHECK(text.find("empty_offset=[") != std::string::npos);
}

// ------------------------------------------------------------------ spmv ----
TEST_CASE("csr5 tile: one segment spanning the whole tile") {  // test_spmv.cpp:78-91
  std::vector<CooEntry> entries;
  for (index_t c = 0; c < 64; ++c) entries.push_back({0, c, static_cast<double>(c + 1)});
  const CsrMatrix a = coo_to_csr(std::move(entries), 1, 64);
  const Csr5Matrix a5 = csr_to_csr5(a, TuningParams{.omega = 32, .sigma = 2});
  const DenseVector x(64, 1.0);
  SpmvWorkspace ws;
  const auto contributions = spmv_csr5_tile(a5, 0, x, ws);
  REQUIRE(contributions.size() == 1);
  CHECK(contributions[0].row == 0);
  CHECK(contributions[0].accumulate);
  CHECK(contributions[0].value == doctest::Approx(2080.0));
}

TEST_CASE("csr5 tile: every entry its own row") {  // test_spmv.cpp:93-105
  std::vector<CooEntry> entries;
  for (index_t i = 0; i < 64; ++i) entries.push_back({i, 0, static_cast<double>(i + 1)});
  const CsrMatrix a = coo_to_csr(std::move(entries), 64, 1);
  const Csr5Matrix a5 = csr_to_csr5(a, TuningParams{.omega = 32, .sigma = 2});
  const DenseVector x{1.0};
  SpmvWorkspace ws;
  const auto contributions = spmv_csr5_tile(a5, 0, x, ws);
  CHECK(contributions.size() == 64);  // one per head
  std::map<index_t, double> by_row;
  for (const auto& c : contributions) by_row[c.row] += c.value;
  for (index_t i = 0; i < 64; ++i) CHECK(by_row[i] == doctest::Approx(double(i + 1)));
}

TEST_CASE("csr5 tile: contribution accounting matches the head count") {  // test_spmv.cpp:107-143
  std::mt19937_64 rng(47);
  for (int trial = 0; trial < 30; ++trial) {
    const index_t m = 1 + static_cast<index_t>(rng() % 120);
    const index_t n = 1 + static_cast<index_t>(rng() % 80);
    const CsrMatrix a = random_csr(rng, m, n, 128 + static_cast<index_t>(rng() % 800));
    const Csr5Matrix a5 = csr_to_csr5(a, TuningParams{.omega = 32, .sigma = 4});
    const DenseVector x = random_x(rng, n);
    SpmvWorkspace ws;
    const CsrMatrix sub = csr5_to_csr(a5);
    for (index_t tid = 0; tid < a5.p_complete; ++tid) {
      const TileDescriptor d = a5.descriptor(tid);
      index_t heads = 0;
      for (auto b : d.bit_flag) heads += b;
      const auto contributions = spmv_csr5_tile(a5, tid, x, ws);
      CHECK(static_cast<index_t>(contributions.size()) == heads);
      const index_t lo = tid * a5.omega() * a5.sigma();
      const index_t hi = lo + a5.omega() * a5.sigma();
      std::map<index_t, double> expect;
      for (index_t r = 0; r < sub.m; ++r) {
        double s = 0.0;
        for (index_t k = std::max(lo, sub.row_ptr[r]); k < std::min(hi, sub.row_ptr[r + 1]); ++k)
          s += sub.val[k] * x[static_cast<std::size_t>(sub.col_idx[k])];
        if (std::max(lo, sub.row_ptr[r]) < std::min(hi, sub.row_ptr[r + 1])) expect[r] = s;
      }
      std::map<index_t, double> got;
      for (const auto& c : contributions) got[c.row] += c.value;
      REQUIRE(got.size() == expect.size());
      for (const auto& [row, v] : expect) {
        REQUIRE(got.contains(row));
        CHECK(got[row] == doctest::Approx(v).epsilon(1e-12));
      }
    }
  }
}

TEST_CASE("csr5: tail-only matrix equals csr-scalar") {  // test_spmv.cpp:145-151
  const CsrMatrix a = coo_to_csr({{1, 0, 2.0}, {3, 1, 4.0}}, 5, 2);
  const Csr5Matrix a5 = csr_to_csr5(a, TuningParams{.omega = 32, .sigma = 4});
  CHECK(a5.p_complete == 0);
  const DenseVector x{1.0, 1.0};
  CHECK(spmv_csr5(a5, x) == spmv_csr_scalar(a, x));
}

TEST_CASE("csr5 equals the oracle across tile shapes and edge shapes") {  // test_spmv.cpp:153-171
  std::mt19937_64 rng(53);
  for (index_t sigma : {1, 2, 4, 12, 16, 27, 48}) {
    for (int trial = 0; trial < 10; ++trial) {
      const index_t m = 1 + static_cast<index_t>(rng() % 150);
      const index_t n = 1 + static_cast<index_t>(rng() % 150);
      const CsrMatrix a = random_csr(rng, m, n, static_cast<index_t>(rng() % 4000));
      const DenseVector x = random_x(rng, n);
      const Csr5Matrix a5 = csr_to_csr5(a, TuningParams{.omega = 32, .sigma = sigma});
      const DenseVector ref = dense_spmv_oracle(a, x);
      check_close(spmv_csr5(a5, x, SpmvMode::deterministic), ref);
      check_close(spmv_csr5(a5, x, SpmvMode::atomic), ref);
      check_close(spmv_csr_segsum(a, x), ref);
    }
  }
}

TEST_CASE("csr5 handles hard shapes") {  // test_spmv.cpp:173-203
  const TuningParams params{.omega = 32, .sigma = 4};
  const DenseVector x1{1.0};
  std::mt19937_64 rng(67);
  SUBCASE("m = 1, wide row") {
    const CsrMatrix a = dense_block(1, 1000);
    const DenseVector x = random_x(rng, 1000);
    check_close(spmv_csr5(csr_to_csr5(a, params), x), dense_spmv_oracle(a, x));
  }
  SUBCASE("n = 1, tall column") {
    const CsrMatrix a = dense_block(1000, 1);
    check_close(spmv_csr5(csr_to_csr5(a, params), x1), dense_spmv_oracle(a, x1));
  }
  SUBCASE("all rows empty") {
    const CsrMatrix a = coo_to_csr({}, 7, 7);
    const DenseVector y = spmv_csr5(csr_to_csr5(a, params), DenseVector(7, 1.0));
    CHECK(y == DenseVector(7, 0.0));
  }
  SUBCASE("one row holds 30% of the nonzeros") {
    std::vector<CooEntry> e;
    for (index_t c = 0; c < 600; ++c) e.push_back({17, c, 1.0 + 0.001 * static_cast<double>(c)});
    for (index_t k = 0; k < 1400; ++k)
      e.push_back({static_cast<index_t>(rng() % 50), static_cast<index_t>(rng() % 2000), 0.75});
    const CsrMatrix a = coo_to_csr(std::move(e), 50, 2000);
    const DenseVector x = random_x(rng, 2000);
    check_close(spmv_csr5(csr_to_csr5(a, params), x), dense_spmv_oracle(a, x));
  }
  SUBCASE("nnz an exact tile multiple") {
    const CsrMatrix a = dense_block(16, 16);
    CHECK(a.nnz() % 128 == 0);
    const DenseVector x = random_x(rng, 16);
    check_close(spmv_csr5(csr_to_csr5(a, params), x), dense_spmv_oracle(a, x));
  }
}

TEST_CASE("csr5 deterministic mode is bit-identical across runs and host threads") {
  std::mt19937_64 rng(59);
  const CsrMatrix a = random_csr(rng, 500, 300, 20000);
  const Csr5Matrix a5 = csr_to_csr5(a, TuningParams{});
  const DenseVector x = random_x(rng, 300);
  const DenseVector first = spmv_csr5(a5, x, SpmvMode::deterministic);
  for (int threads : {1, 2, 8}) {
    std::vector<DenseVector> ys(static_cast<std::size_t>(threads));
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&, t] { ys[static_cast<std::size_t>(t)] = spmv_csr5(a5, x); });
    for (auto& th : pool) th.join();
    for (const DenseVector& y : ys)
      CHECK(std::memcmp(first.data(), y.data(), y.size() * sizeof(double)) == 0);
  }
}

TEST_CASE("csr5 scaling by a power of two is exact") {  // test_spmv.cpp:232-242
  std::mt19937_64 rng(61);
  const CsrMatrix a = random_csr(rng, 40, 40, 400);
  const DenseVector x = random_x(rng, 40);
  DenseVector x8(x);
  for (double& v : x8) v *= 8.0;
  const Csr5Matrix a5 = csr_to_csr5(a, TuningParams{.omega = 32, .sigma = 4});
  const DenseVector y = spmv_csr5(a5, x);
  const DenseVector y8 = spmv_csr5(a5, x8);
  for (std::size_t i = 0; i < y.size(); ++i) CHECK(y8[i] == 8.0 * y[i]);
}

TEST_CASE("csr5 with 64-bit descriptor words") {  // test_spmv.cpp:244-254
  // sigma = 40 pushes a column past 32 bits (40 + 11 + 5 = 56)
  std::mt19937_64 rng(71);
  const CsrMatrix a = random_csr(rng, 80, 60, 4000);
  const TuningParams params{.omega = 32, .sigma = 40};
  const Csr5Matrix a5 = csr_to_csr5(a, params);
  CHECK(a5.layout.word_bits == 64);
  CHECK(csr5_to_csr(a5) == a);
  const DenseVector x = random_x(rng, 60);
  check_close(spmv_csr5(a5, x), dense_spmv_oracle(a, x));
}

TEST_CASE("csr5 rejects dimension mismatches and bad tile ids") {  // test_spmv.cpp:256-262
  const CsrMatrix a = coo_to_csr({{0, 0, 1.0}}, 2, 3);
  const Csr5Matrix a5 = csr_to_csr5(a, TuningParams{});
  CHECK_THROWS_AS(spmv_csr5(a5, DenseVector(2, 1.0)), std::invalid_argument);
  SpmvWorkspace ws;
  CHECK_THROWS_AS(spmv_csr5_tile(a5, 0, DenseVector(3, 1.0), ws), std::invalid_argument);
}

int main() { return mini::run_all(); }
