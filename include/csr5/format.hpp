// csr5/format.hpp -- drop-in for the reference's format.hpp (format.hpp:1-190):
// the tile-pointer encoding, the index helpers, Csr5Matrix, csr_to_csr5,
// csr5_to_csr and dump_format, over the GPU library (include/csr5g.h).
//
// Csr5Matrix keeps the reference's public members.  The scalars are filled
// at construction; the array members (tile_ptr, tile_desc, empty_offset_ptr,
// empty_offset, row_ptr, col_idx, val) are read-only views of the device
// arrays, copied to the host once, on first access -- an SpMV never touches
// them.  Copies of a Csr5Matrix share one immutable device handle, released
// with the last copy (the reference's value semantics, format.hpp:130).
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <ostream>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "csr5/csr.hpp"
#include "csr5/descriptor.hpp"
#include "csr5/tuning.hpp"

namespace csr5 {

/// Raw tile pointer word (format.hpp:14-22): MSB of the word = the tile's row
/// range holds an empty row; the rest = the tile's first row.
struct TilePointer {
  std::uint64_t raw = 0;

  bool operator==(const TilePointer&) const = default;
};

/// 32 while row indices fit in 31 bits, otherwise 64 (format.cpp:18-20).
/// The GPU build supports the 32-bit case (m < 2^31) and rejects larger m
/// with std::out_of_range.
inline int tile_ptr_bits_for_rows(index_t m) { return m < (index_t{1} << 31) ? 32 : 64; }

inline std::uint64_t encode_tile_ptr(index_t row, bool empty_rows, int bits) {
  const std::uint64_t msb = std::uint64_t{1} << (bits - 1);
  if (static_cast<std::uint64_t>(row) >= msb)
    throw std::invalid_argument("tile_ptr: row index does not fit in " + std::to_string(bits - 1) +
                                " bits");
  return static_cast<std::uint64_t>(row) | (empty_rows ? msb : 0);
}
inline index_t decode_tile_ptr_row(std::uint64_t raw, int bits) {
  return static_cast<index_t>(raw & ((std::uint64_t{1} << (bits - 1)) - 1));
}
inline bool decode_tile_ptr_flag(std::uint64_t raw, int bits) { return (raw >> (bits - 1)) & 1u; }

/// Position of (column i, depth j) of tile tid before (logical) and after
/// (physical) the transposition (format.hpp:35-42).
constexpr index_t tile_logical_index(index_t tid, index_t omega, index_t sigma, index_t i,
                                     index_t j) {
  return (tid * omega + i) * sigma + j;
}
constexpr index_t tile_physical_index(index_t tid, index_t omega, index_t sigma, index_t i,
                                      index_t j) {
  return (tid * sigma + j) * omega + i;
}

/// The row owning nonzero g: the last row r with row_ptr[r] <= g, clamped to
/// [0, m-1] (format.cpp:42-50).
inline index_t row_of_nonzero(std::span<const index_t> row_ptr, index_t g) {
  const index_t m = static_cast<index_t>(row_ptr.size()) - 1;
  if (m <= 0) return 0;
  const index_t past = std::upper_bound(row_ptr.begin(), row_ptr.end(), g) - row_ptr.begin();
  return std::clamp<index_t>(past - 1, 0, m - 1);
}

/// Tile transposition of the complete omega*sigma blocks, tail untouched
/// (format.hpp:76-103): host data movement helpers, as in the reference.
template <class T>
void transpose_tiles_forward(std::span<T> data, index_t omega, index_t sigma) {
  const std::size_t w = static_cast<std::size_t>(omega), h = static_cast<std::size_t>(sigma);
  if (w * h <= 1) return;
  std::vector<T> block(w * h);
  for (std::size_t off = 0; off + w * h <= data.size(); off += w * h) {
    for (std::size_t q = 0; q < w * h; ++q) block[(q % h) * w + q / h] = data[off + q];
    std::copy(block.begin(), block.end(), data.begin() + static_cast<std::ptrdiff_t>(off));
  }
}
template <class T>
void transpose_tiles_inverse(std::span<T> data, index_t omega, index_t sigma) {
  const std::size_t w = static_cast<std::size_t>(omega), h = static_cast<std::size_t>(sigma);
  if (w * h <= 1) return;
  std::vector<T> block(w * h);
  for (std::size_t off = 0; off + w * h <= data.size(); off += w * h) {
    for (std::size_t q = 0; q < w * h; ++q) block[q] = data[off + (q % h) * w + q / h];
    std::copy(block.begin(), block.end(), data.begin() + static_cast<std::ptrdiff_t>(off));
  }
}

/// Word array at the narrowest configured width (format.hpp:106-124).  Either
/// owns its words (the reference's constructor) or views a handle's device
/// array (Csr5Matrix::tile_ptr / tile_desc).
class PackedWords {
 public:
  PackedWords() = default;
  PackedWords(std::span<const std::uint64_t> words, int word_bits) : bits_(word_bits) {
    if (word_bits != 32 && word_bits != 64)
      throw std::invalid_argument("PackedWords: word width must be 32 or 64");
    if (word_bits == 32)
      for (std::uint64_t v : words)
        if (v >> 32) throw std::invalid_argument("PackedWords: value does not fit in 32 bits");
    own_.assign(words.begin(), words.end());
    count_ = own_.size();
  }
  PackedWords(detail::HostArray<std::uint64_t> view, std::size_t count, int word_bits)
      : bits_(word_bits), count_(count), view_(std::move(view)), lazy_(true) {}

  std::uint64_t operator[](std::size_t i) const { return words()[i]; }
  std::size_t size() const { return count_; }
  int word_bits() const { return bits_; }
  std::size_t byte_size() const { return count_ * static_cast<std::size_t>(bits_ / 8); }
  bool operator==(const PackedWords& o) const { return bits_ == o.bits_ && words() == o.words(); }

 private:
  const std::vector<std::uint64_t>& words() const { return lazy_ ? view_.vec() : own_; }
  int bits_ = 32;
  std::size_t count_ = 0;
  std::vector<std::uint64_t> own_;
  detail::HostArray<std::uint64_t> view_;
  bool lazy_ = false;
};

/// The five-array tiled format (format.hpp:126-176), resident on the GPU.
struct Csr5Matrix {
  index_t m = 0;
  index_t n = 0;
  index_t nnz = 0;
  TuningParams params;

  index_t p = 0;           // tile count, ceil(nnz / (omega * sigma))
  index_t p_complete = 0;  // floor(nnz / (omega * sigma))
  index_t tail_len = 0;    // nnz mod (omega * sigma)

  int tile_ptr_bits = 32;
  DescriptorLayout layout;

  PackedWords tile_ptr;   // p + 1 words
  PackedWords tile_desc;  // p_complete * omega words

  detail::HostArray<index_t> empty_offset_ptr;  // p_complete + 1
  detail::HostArray<index_t> empty_offset;
  detail::HostArray<index_t> row_ptr;  // m + 1, identical to the source CSR
  detail::HostArray<index_t> col_idx;  // tile-transposed, tail unchanged
  detail::HostArray<double> val;

  index_t omega() const { return params.omega; }
  index_t sigma() const { return params.sigma; }
  index_t tile_row(index_t tid) const {
    return decode_tile_ptr_row(tile_ptr[static_cast<std::size_t>(tid)], tile_ptr_bits);
  }
  bool tile_has_empty_rows(index_t tid) const {
    return decode_tile_ptr_flag(tile_ptr[static_cast<std::size_t>(tid)], tile_ptr_bits);
  }
  /// Unpacked descriptor of complete tile tid (format.cpp:152-157).
  TileDescriptor descriptor(index_t tid) const {
    std::vector<std::uint64_t> w(static_cast<std::size_t>(omega()));
    for (index_t i = 0; i < omega(); ++i)
      w[static_cast<std::size_t>(i)] = tile_desc[static_cast<std::size_t>(tid * omega() + i)];
    return unpack_tile_descriptor(w, layout);
  }
  std::size_t metadata_bytes() const { return tile_ptr.byte_size() + tile_desc.byte_size(); }
  static std::size_t csr_bytes(index_t m, index_t nnz, int index_bits) {
    const std::size_t ib = static_cast<std::size_t>(index_bits / 8);
    return static_cast<std::size_t>(nnz) * (ib + sizeof(double)) +
           static_cast<std::size_t>(m + 1) * ib;
  }

  // ---- GPU extras (not in the reference) ----
  csr5g_matrix handle() const { return dev_ ? dev_->h : nullptr; }
  const csr5g_info& info() const {
    static const csr5g_info none{};
    return dev_ ? dev_->info : none;
  }

  /// Wraps a built handle (takes ownership).
  static Csr5Matrix from_handle(csr5g_matrix h, const TuningParams& params) {
    Csr5Matrix r;
    r.dev_ = std::make_shared<detail::Device>(h);
    const csr5g_info& i = r.dev_->info;
    r.m = i.m;
    r.n = i.n;
    r.nnz = i.nnz;
    r.params = params;
    r.params.sigma = i.sigma;
    r.p = i.p;
    r.p_complete = i.p_complete;
    r.tail_len = i.tail_len;
    r.tile_ptr_bits = i.tile_ptr_bits;
    r.layout = DescriptorLayout{i.omega, i.sigma, i.y_offset_bits, i.seg_offset_bits, i.word_bits};
    using D = detail::Device;
    r.tile_ptr = PackedWords(detail::HostArray<std::uint64_t>(r.dev_, &D::tile_ptr),
                             static_cast<std::size_t>(i.tile_ptr_len), i.tile_ptr_bits);
    r.tile_desc = PackedWords(detail::HostArray<std::uint64_t>(r.dev_, &D::tile_desc),
                              static_cast<std::size_t>((i.tile_end - i.tile_begin) * i.omega),
                              i.word_bits);
    r.empty_offset_ptr = detail::HostArray<index_t>(r.dev_, &D::empty_offset_ptr);
    r.empty_offset = detail::HostArray<index_t>(r.dev_, &D::empty_offset);
    r.row_ptr = detail::HostArray<index_t>(r.dev_, &D::row_ptr);
    r.col_idx = detail::HostArray<index_t>(r.dev_, &D::col_idx);
    r.val = detail::HostArray<double>(r.dev_, &D::val);
    return r;
  }

 private:
  std::shared_ptr<detail::Device> dev_;
};

/// format.cpp:165-252: the CSR staged to the current CUDA device and
/// converted there (csr5g_build_host).  The input is not modified; `parallel`
/// is accepted for source compatibility (the GPU build is always parallel and
/// deterministic).  omega must be 32 (one warp lane per tile column).
inline Csr5Matrix csr_to_csr5(const CsrMatrix& a, const TuningParams& params,
                              bool parallel = true) {
  (void)parallel;
  params.validate();
  if (static_cast<index_t>(a.row_ptr.size()) != a.m + 1)
    throw std::runtime_error("csr: row_ptr has size " + std::to_string(a.row_ptr.size()) +
                             ", expected " + std::to_string(a.m + 1));
  if (static_cast<index_t>(a.col_idx.size()) != a.nnz() ||
      static_cast<index_t>(a.val.size()) != a.nnz())
    throw std::runtime_error("csr: col_idx/val size does not match row_ptr[m]");
  const csr5g_params p{params.omega, params.sigma, params.r, params.s, params.t, params.u};
  csr5g_matrix h = nullptr;
  detail::check(csr5g_build_host(-1, a.m, a.n, a.nnz(), a.row_ptr.data(), a.col_idx.data(),
                                 a.val.data(), &p, &h));
  return Csr5Matrix::from_handle(h, params);
}

/// format.cpp:254-265: undoes the transposition (on the device) and returns
/// the source CSR bit for bit; validated like the reference's.
inline CsrMatrix csr5_to_csr(const Csr5Matrix& a5) {
  CsrMatrix a;
  a.m = a5.m;
  a.n = a5.n;
  if (a5.handle()) {
    a.row_ptr.resize(static_cast<std::size_t>(a5.m) + 1);
    detail::check(csr5g_export_row_ptr(a5.handle(), a.row_ptr.data()));
    a.col_idx.resize(static_cast<std::size_t>(a5.nnz));
    a.val.resize(static_cast<std::size_t>(a5.nnz));
    detail::check(csr5g_to_csr_host(a5.handle(), a.col_idx.data(), a.val.data()));
  } else {
    a.row_ptr.assign(static_cast<std::size_t>(a5.m) + 1, 0);
  }
  validate(a);
  return a;
}

/// Text dump of the tile metadata, one tile per line (format.cpp:267-305;
/// byte-identical output, tests/test_gpu_dump.py).
inline void dump_format(const Csr5Matrix& a5, std::ostream& out) {
  out << "csr5 m=" << a5.m << " n=" << a5.n << " nnz=" << a5.nnz << " omega=" << a5.omega()
      << " sigma=" << a5.sigma() << " tiles=" << a5.p << " complete=" << a5.p_complete
      << " tail=" << a5.tail_len << " tile_ptr_bits=" << a5.tile_ptr_bits
      << " desc_word_bits=" << a5.layout.word_bits << " metadata_bytes=" << a5.metadata_bytes()
      << " empty_offset_entries=" << a5.empty_offset.size() << '\n';
  auto list = [&out](const char* label, auto first, auto last) {
    out << ' ' << label << "=[";
    for (auto it = first; it != last; ++it) out << (it == first ? "" : ",") << *it;
    out << ']';
  };
  for (index_t t = 0; t < a5.p; ++t) {
    out << "tile " << t << ": row=" << a5.tile_row(t) << " empty=" << (a5.tile_has_empty_rows(t) ? 1 : 0);
    if (t >= a5.p_complete) {
      out << " tail nnz=" << a5.tail_len << '\n';
      continue;
    }
    const TileDescriptor d = a5.descriptor(t);
    list("y_offset", d.y_offset.begin(), d.y_offset.end());
    list("seg_offset", d.seg_offset.begin(), d.seg_offset.end());
    out << " bit_flag=[";
    const std::size_t h = static_cast<std::size_t>(a5.sigma());
    for (std::size_t q = 0; q < d.bit_flag.size(); ++q)
      out << (q && q % h == 0 ? "," : "") << (d.bit_flag[q] ? '1' : '0');
    out << ']';
    if (a5.tile_has_empty_rows(t)) {
      const auto b = a5.empty_offset.begin();
      list("empty_offset", b + a5.empty_offset_ptr[static_cast<std::size_t>(t)],
           b + a5.empty_offset_ptr[static_cast<std::size_t>(t) + 1]);
    }
    out << '\n';
  }
}

// ---- the construction steps (format.hpp:44-75), for tests and tooling ----

/// All p + 1 tile pointers, from a GPU build at (omega, sigma).
inline std::vector<TilePointer> generate_tile_ptr(const CsrMatrix& a, index_t omega, index_t sigma) {
  const Csr5Matrix a5 = csr_to_csr5(a, TuningParams{.omega = omega, .sigma = sigma});
  std::vector<TilePointer> out(a5.tile_ptr.size());
  for (std::size_t i = 0; i < out.size(); ++i) out[i].raw = a5.tile_ptr[i];
  return out;
}

/// bit_flag of complete tile tid, from a GPU build at (omega, sigma).
inline std::vector<std::uint8_t> generate_bit_flag(const CsrMatrix& a, index_t tid, index_t omega,
                                                   index_t sigma) {
  return csr_to_csr5(a, TuningParams{.omega = omega, .sigma = sigma}).descriptor(tid).bit_flag;
}

/// y_offset (exclusive scan of per-column head counts) and seg_offset (the
/// run of headless columns right of each head-bearing column) of a given
/// bit_flag (format.cpp:102-121 semantics).
inline std::pair<std::vector<index_t>, std::vector<index_t>> generate_y_and_seg_offset(
    std::span<const std::uint8_t> bit_flag, index_t omega, index_t sigma) {
  const std::size_t w = static_cast<std::size_t>(omega), h = static_cast<std::size_t>(sigma);
  if (bit_flag.size() != w * h)
    throw std::invalid_argument("generate_y_and_seg_offset: bit_flag size mismatch");
  std::vector<index_t> y(w, 0), seg(w, 0);
  std::vector<bool> has(w, false);
  index_t heads = 0;
  for (std::size_t c = 0; c < w; ++c) {
    y[c] = heads;
    for (std::size_t d = 0; d < h; ++d) heads += bit_flag[c * h + d] ? 1 : 0;
    has[c] = heads != y[c];
  }
  for (std::size_t c = 0; c < w; ++c) {
    if (!has[c]) continue;
    std::size_t e = c + 1;
    while (e < w && !has[e]) ++e;
    seg[c] = static_cast<index_t>(e - c - 1);
  }
  return {std::move(y), std::move(seg)};
}

/// Row offsets (row_of_nonzero - tile_row) of every head of `bit_flag`, in
/// column-major head order (format.cpp:123-136 semantics).
inline std::vector<index_t> generate_empty_offset(const CsrMatrix& a, index_t tid, index_t tile_row,
                                                  std::span<const std::uint8_t> bit_flag,
                                                  index_t omega, index_t sigma) {
  std::vector<index_t> out;
  const std::span<const index_t> rp(a.row_ptr);
  const index_t base = tid * omega * sigma;
  for (std::size_t q = 0; q < bit_flag.size(); ++q)
    if (bit_flag[q]) out.push_back(row_of_nonzero(rp, base + static_cast<index_t>(q)) - tile_row);
  return out;
}

}  // namespace csr5
