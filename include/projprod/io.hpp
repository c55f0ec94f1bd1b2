#pragma once
// PT3 container I/O (proj/include/projprod/io.hpp:11-30) over the engine's
// ppc_pt3_* C-ABI.
//
//   offset  size  field
//   0       4     magic "PT3\0"
//   4       4     u32 version (= 1)
//   8       1     u8 dtype (1 = float64 little-endian)
//   9       1     u8 field flags (= 0)
//   10      2     padding (zero)
//   12      24    u64 n1, n2, n3
//   36      ...   payload: 8*n1*n2*n3 bytes, mode-1 fastest
#include <cstdint>
#include <filesystem>

#include "projprod/tensor.hpp"

namespace projprod {

inline constexpr std::uint32_t kPt3Version = 1;

void write_pt3(const std::filesystem::path& path, const Tensor3& A);
Tensor3 read_pt3(const std::filesystem::path& path);

// Matrix convenience wrappers over the degenerate n3 = 1 form.
void write_pt3_matrix(const std::filesystem::path& path, const Matrix& M);
Matrix read_pt3_matrix(const std::filesystem::path& path);

}  // namespace projprod
