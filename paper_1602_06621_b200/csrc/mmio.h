// mmio.h -- Matrix Market and binary CSR files (host side; mmio.cpp).
#pragma once

#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

namespace eqb {
namespace mm {

struct Matrix {
  bool dense = false;
  int64_t m = 0, n = 0, nnz = 0;
  std::vector<int64_t> row, col, line;  // coordinate entries (0-based) and their lines
  std::vector<double> val;
  std::vector<double> dense_rowmajor;   // array format, converted to row-major
};

// read_matrix_market (src/matrix_market.cpp:63-198); throws std::runtime_error
// "matrix market: line N: ..." exactly as the reference does
void parse(const char* data, size_t len, Matrix& out);
void read_file(const std::string& path, std::string& buf);
void write_coordinate(const std::string& path, int64_t m, int64_t n, const int64_t* rp,
                      const int32_t* col, const double* val);
void write_array(const std::string& path, int64_t m, int64_t n, const double* rowmajor);

void write_binary(const std::string& path, int64_t m, int64_t n, bool dense, const int64_t* rp,
                  const int32_t* col, const double* val, const double* rowmajor);
void read_binary_header(FILE* f, const std::string& path, int64_t hdr[4]);
void read_exact(FILE* f, void* dst, size_t size, size_t count, const std::string& path);

}  // namespace mm
}  // namespace eqb
