// csr5/descriptor.hpp -- drop-in for the reference's descriptor.hpp
// (descriptor.cpp:17-88): the tile descriptor's logical view and its packed
// bit layout.  Pure bit-field helpers on one descriptor; the GPU converter
// packs the same layout (convert.cu, k_desc_transpose).
#pragma once

#include <bit>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "csr5/csr.hpp"

namespace csr5 {

/// Logical view of one complete tile's descriptor (descriptor.hpp:11-24).
struct TileDescriptor {
  std::vector<index_t> y_offset;       // omega entries
  std::vector<index_t> seg_offset;     // omega entries
  std::vector<std::uint8_t> bit_flag;  // omega * sigma entries, column-major

  bool operator==(const TileDescriptor&) const = default;
};

/// Number of bits needed to represent every value in [0, v).
inline int ceil_log2(index_t v) {
  if (v < 1) throw std::invalid_argument("ceil_log2: argument must be >= 1");
  return std::bit_width(static_cast<std::uint64_t>(v) - 1);
}

/// Bit-field layout of one packed descriptor column, most significant first
/// [y_offset | seg_offset | bit_flag]; depth j's flag at bit sigma - 1 - j.
struct DescriptorLayout {
  index_t omega = 0;
  index_t sigma = 0;
  int y_offset_bits = 0;
  int seg_offset_bits = 0;
  int word_bits = 32;

  int column_bits() const { return y_offset_bits + seg_offset_bits + static_cast<int>(sigma); }

  bool operator==(const DescriptorLayout&) const = default;
};

/// descriptor.cpp:22-36, evaluated by the library (csr5g_layout: the same
/// rule, the same std::invalid_argument texts).
inline DescriptorLayout make_descriptor_layout(index_t omega, index_t sigma) {
  std::int32_t yb = 0, sb = 0, wb = 0;
  detail::check(csr5g_layout(omega, sigma, &yb, &sb, &wb));
  return DescriptorLayout{omega, sigma, yb, sb, wb};
}

namespace detail {
// Field positions of one packed column: [y | seg | flags], flags lowest.
struct Fields {
  int flag_bits, seg_shift, y_shift;
  std::uint64_t seg_max, y_max;
  explicit Fields(const DescriptorLayout& l)
      : flag_bits(static_cast<int>(l.sigma)),
        seg_shift(static_cast<int>(l.sigma)),
        y_shift(static_cast<int>(l.sigma) + l.seg_offset_bits),
        seg_max(l.seg_offset_bits >= 64 ? ~0ull : (1ull << l.seg_offset_bits) - 1),
        y_max(l.y_offset_bits >= 64 ? ~0ull : (1ull << l.y_offset_bits) - 1) {}
};
}  // namespace detail

/// descriptor.cpp:38-62 semantics: one word per column; std::invalid_argument
/// on mismatched sizes or a field that does not fit its bits.
inline std::vector<std::uint64_t> pack_tile_descriptor(const TileDescriptor& d,
                                                       const DescriptorLayout& layout) {
  const std::size_t w = static_cast<std::size_t>(layout.omega);
  const std::size_t h = static_cast<std::size_t>(layout.sigma);
  if (d.y_offset.size() != w || d.seg_offset.size() != w || d.bit_flag.size() != w * h)
    throw std::invalid_argument("pack_tile_descriptor: array sizes do not match the layout");
  const detail::Fields f(layout);
  std::vector<std::uint64_t> out;
  out.reserve(w);
  for (std::size_t col = 0; col < w; ++col) {
    const auto yv = static_cast<std::uint64_t>(d.y_offset[col]);
    const auto sv = static_cast<std::uint64_t>(d.seg_offset[col]);
    if (yv > f.y_max || sv > f.seg_max)
      throw std::invalid_argument("pack_tile_descriptor: field overflow in column " +
                                  std::to_string(col));
    std::uint64_t flags = 0;  // depth 0 ends up in the highest flag bit
    for (std::size_t dep = 0; dep < h; ++dep) flags = (flags << 1) | (d.bit_flag[col * h + dep] ? 1u : 0u);
    out.push_back((yv << f.y_shift) | (sv << f.seg_shift) | flags);
  }
  return out;
}

/// descriptor.cpp:64-88 semantics: the exact inverse of pack_tile_descriptor.
inline TileDescriptor unpack_tile_descriptor(std::span<const std::uint64_t> words,
                                             const DescriptorLayout& layout) {
  const std::size_t w = static_cast<std::size_t>(layout.omega);
  const std::size_t h = static_cast<std::size_t>(layout.sigma);
  if (words.size() != w)
    throw std::invalid_argument("unpack_tile_descriptor: expected one word per column");
  const detail::Fields f(layout);
  TileDescriptor d;
  d.bit_flag.reserve(w * h);
  for (const std::uint64_t word : words) {
    d.y_offset.push_back(static_cast<index_t>((word >> f.y_shift) & f.y_max));
    d.seg_offset.push_back(static_cast<index_t>((word >> f.seg_shift) & f.seg_max));
    for (std::size_t dep = h; dep-- > 0;) d.bit_flag.push_back(static_cast<std::uint8_t>((word >> dep) & 1u));
  }
  return d;
}

}  // namespace csr5
