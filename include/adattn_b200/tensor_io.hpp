// adattn_b200/tensor_io.hpp -- drop-in for the reference's ATN1 tensor files
// (/root/reference/proj/include/adattn/tensor_io.hpp:9-31, src/tensor_io.cpp:39-112):
// magic "ATN1", dtype byte (0 = f32, 1 = f64), rank u32 (1..3), rank u32 dims,
// row-major little-endian payload.  Parse errors throw std::runtime_error with
// the byte offset; writes go to "<path>.tmp" and are renamed into place.
// Implemented in libadattn_b200.so (csrc/io.cu); the same code backs the C-ABI
// adattn_b200_tensor_* entry points.
#pragma once

#include <cstdint>
#include <filesystem>
#include <vector>

namespace adattn {

enum class Dtype : uint8_t { kF32 = 0, kF64 = 1 };

struct Tensor {
  Dtype dtype = Dtype::kF64;
  std::vector<uint32_t> dims;
  std::vector<double> values;

  size_t count() const {
    size_t c = 1;
    for (uint32_t d : dims) c *= d;
    return c;
  }
};

Tensor load_tensor(const std::filesystem::path& path);
void save_tensor(const Tensor& t, const std::filesystem::path& path);

}  // namespace adattn
