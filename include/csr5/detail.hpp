// csr5/detail.hpp -- plumbing under the csr5:: drop-in headers: status ->
// exception mapping and the shared device handle behind Csr5Matrix.
// Not part of the reference API.
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "csr5g.h"

namespace csr5::detail {

// The reference throws std::invalid_argument for argument / layout errors,
// std::out_of_range for range errors and std::runtime_error otherwise; the
// library's status codes map onto the same types with the same text.
inline void check(int rc) {
  if (rc == CSR5G_OK) return;
  const std::string msg = csr5g_last_error();
  if (rc == CSR5G_EINVAL) throw std::invalid_argument(msg);
  if (rc == CSR5G_ERANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}

// One built handle (device arrays owned by libcsr5g), shared read-only by
// every copy of a Csr5Matrix (the reference's value type is immutable after
// construction).  Host copies of the arrays are fetched once, on
// first access to a Csr5Matrix array member.
struct Device {
  csr5g_matrix h = nullptr;
  csr5g_info info{};
  std::once_flag fetched;
  std::vector<std::uint64_t> tile_ptr, tile_desc;
  std::vector<std::int64_t> empty_offset_ptr, empty_offset, row_ptr, col_idx;
  std::vector<double> val;

  explicit Device(csr5g_matrix handle) : h(handle) { check(csr5g_info_get(h, &info)); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  ~Device() {
    if (h) csr5g_release(h);
  }

  void fetch() {
    std::call_once(fetched, [this] {
      const std::int64_t pcs = info.tile_end - info.tile_begin;
      tile_ptr.resize((std::size_t)info.tile_ptr_len);
      tile_desc.resize((std::size_t)(pcs * info.omega));
      empty_offset_ptr.resize((std::size_t)(pcs + 1));
      empty_offset.resize((std::size_t)info.empty_offset_len);
      col_idx.resize((std::size_t)info.nnz_held);
      val.resize((std::size_t)info.nnz_held);
      row_ptr.resize((std::size_t)info.m + 1);
      check(csr5g_export(h, tile_ptr.data(), tile_desc.data(), empty_offset_ptr.data(),
                         empty_offset.data(), col_idx.data(), val.data()));
      check(csr5g_export_row_ptr(h, row_ptr.data()));
    });
  }
};

// A read-only view of one host copy of a device array: the reference's
// std::vector member, materialised on first use.
template <class T>
class HostArray {
 public:
  using value_type = T;
  using const_iterator = typename std::vector<T>::const_iterator;

  HostArray() = default;
  HostArray(std::shared_ptr<Device> d, std::vector<T> Device::*member)
      : d_(std::move(d)), member_(member) {}

  const std::vector<T>& vec() const {
    static const std::vector<T> empty;
    if (!d_) return empty;
    d_->fetch();
    return (*d_).*member_;
  }
  operator const std::vector<T>&() const { return vec(); }  // NOLINT: reference API
  const T& operator[](std::size_t i) const { return vec()[i]; }
  std::size_t size() const { return vec().size(); }
  bool empty() const { return vec().empty(); }
  const T* data() const { return vec().data(); }
  const_iterator begin() const { return vec().begin(); }
  const_iterator end() const { return vec().end(); }
  const T& front() const { return vec().front(); }
  const T& back() const { return vec().back(); }
  friend bool operator==(const HostArray& a, const std::vector<T>& b) { return a.vec() == b; }
  friend bool operator==(const HostArray& a, const HostArray& b) { return a.vec() == b.vec(); }

 private:
  std::shared_ptr<Device> d_;
  std::vector<T> Device::*member_ = nullptr;
};

}  // namespace csr5::detail
