// Dense matrix interchange (reference nystrom.cpp:450-477): u32 rows, u32
// cols, then the entries row by row as doubles.  The reference uses it to
// hand dense factors between runs; here it is also the tier-1 route for the
// oracle's update factors L, R into the device ELS.
#include <cstdio>
#include <cstdint>

#include "matio.hpp"

namespace sbx {

void dump_matrix(const std::string& path, const double* m, i64 rows, i64 cols, i64 ld) {
  require(rows >= 0 && cols >= 0 && rows <= i64(UINT32_MAX) && cols <= i64(UINT32_MAX),
          "dump_matrix: dimensions out of range");
  require(ld >= rows, "dump_matrix: leading dimension smaller than rows");
  std::FILE* fp = std::fopen(path.c_str(), "wb");
  require(fp != nullptr, "dump_matrix: cannot open " + path);
  const std::uint32_t dims[2] = {std::uint32_t(rows), std::uint32_t(cols)};
  bool ok = std::fwrite(dims, sizeof(std::uint32_t), 2, fp) == 2;
  std::vector<double> row(static_cast<size_t>(cols));
  for (i64 i = 0; ok && i < rows; ++i) {
    for (i64 j = 0; j < cols; ++j) row[size_t(j)] = m[i + j * ld];
    ok = std::fwrite(row.data(), sizeof(double), row.size(), fp) == row.size();
  }
  std::fclose(fp);
  require(ok, "dump_matrix: write failed for " + path);
}

HMat load_matrix(const std::string& path) {
  std::FILE* fp = std::fopen(path.c_str(), "rb");
  require(fp != nullptr, "load_matrix: cannot open " + path);
  std::uint32_t dims[2];
  if (std::fread(dims, sizeof(std::uint32_t), 2, fp) != 2) {
    std::fclose(fp);
    throw Error(1, "load_matrix: bad header");
  }
  HMat m(dims[0], dims[1]);
  std::vector<double> row(dims[1]);
  for (std::uint32_t i = 0; i < dims[0]; ++i) {
    if (std::fread(row.data(), sizeof(double), dims[1], fp) != dims[1]) {
      std::fclose(fp);
      throw Error(1, "load_matrix: truncated");
    }
    for (std::uint32_t j = 0; j < dims[1]; ++j) m.a[size_t(i + i64(j) * m.r)] = row[j];
  }
  std::fclose(fp);
  return m;
}

}  // namespace sbx
