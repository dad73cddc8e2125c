// Matrix Market I/O of the drop-in API (include/intgmres/mm_io.hpp) against
// the reference's documented behaviour (proj/core/src/mm_io.cpp): accepted
// inputs, "path:line: message" diagnostics, bit-exact save/load round trip.
// Prints "ok" or the first failure; host-only (no GPU needed).
#include <intgmres/csr.hpp>
#include <intgmres/mm_io.hpp>

#include <cstdio>
#include <cstring>
#include <unistd.h>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

using namespace intgmres;

static std::string tmp_path() { return "/tmp/igm_mm_test_" + std::to_string(::getpid()) + ".mtx"; }
static void write(const std::string& p, const std::string& text) { std::ofstream(p) << text; }

static std::string error_of(const std::string& text) {
  const std::string p = tmp_path();
  write(p, text);
  try {
    load_matrix_market(p);
    return "(no error)";
  } catch (const std::runtime_error& e) {
    const std::string m = e.what();
    return m.substr(m.find(':') + 1);
  }
}

#define EXPECT(cond, what)                          \
  do {                                              \
    if (!(cond)) {                                  \
      std::printf("FAIL: %s\n", what);             \
      return 1;                                     \
    }                                               \
  } while (0)

int main() {
  const std::string p = tmp_path();
  write(p, "%%MatrixMarket matrix coordinate real general\n% c\n\n3 3 4\n1 1 2.5\n3 1 -1\n2 2 4\n1 3 0.5\n");
  CsrMatrixF a = load_matrix_market(p);
  EXPECT(a.n == 3 && a.nnz() == 4, "general: sizes");
  EXPECT((a.row_ptr == std::vector<int>{0, 2, 3, 4}), "general: row_ptr");
  EXPECT((a.col_idx == std::vector<int>{0, 2, 1, 0}), "general: col_idx");
  EXPECT((a.vals == std::vector<double>{2.5, 0.5, 4.0, -1.0}), "general: vals");
  write(p, "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 3\n2 1 -2\n");
  a = load_matrix_market(p);
  EXPECT((a.vals == std::vector<double>{3.0, -2.0, -2.0}) && a.nnz() == 3, "symmetric expansion");
  write(p, "%%MatrixMarket MATRIX Coordinate Integer General\n1 1 1\n1 1 7\n");
  EXPECT(load_matrix_market(p).vals == std::vector<double>{7.0}, "integer field, case-insensitive banner words");
  EXPECT(error_of("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n") ==
             "1: unsupported field type 'complex'", "complex");
  EXPECT(error_of("%%MatrixMarket matrix array real general\n1 1\n1\n") == "1: only coordinate matrices are supported",
         "array");
  EXPECT(error_of("hello\n1 1 1\n1 1 1\n") == "1: missing MatrixMarket banner", "banner");
  EXPECT(error_of("%%MatrixMarket matrix coordinate real skew-symmetric\n1 1 1\n1 1 1\n") ==
             "1: unsupported symmetry 'skew-symmetric'", "symmetry");
  EXPECT(error_of("%%MatrixMarket matrix coordinate real general\n3 2 1\n1 1 1.0\n") == "2: matrix must be square",
         "square");
  EXPECT(error_of("%%MatrixMarket matrix coordinate real general\n2 2 2\n2 1 1.0\n2 1 2.0\n") == "4: duplicate entry",
         "duplicate");
  EXPECT(error_of("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\nx y z\n") == "4: malformed entry",
         "malformed");
  EXPECT(error_of("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n1 3 1.0\n") ==
             "4: index out of range", "range");
  EXPECT(error_of("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n2 2 1.0\n") ==
             "4: fewer entries than declared (2 of 3)", "fewer");
  EXPECT(error_of("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n2 2 1.0\n") ==
             "4: more entries than declared", "more");
  EXPECT(error_of("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 2 1.0\n") ==
             "3: symmetric file stores only the lower triangle", "upper triangle");
  EXPECT(error_of("%%MatrixMarket matrix coordinate real general\n0 0 0\n") == "2: matrix must be non-empty", "empty");
  EXPECT(error_of("%%MatrixMarket matrix coordinate real general\n% only\n") == "2: missing size line", "no size");
  try {
    load_matrix_market("/nonexistent/nowhere.mtx");
    EXPECT(false, "missing file");
  } catch (const std::runtime_error& e) {
    EXPECT(std::string(e.what()) == "/nonexistent/nowhere.mtx: cannot open file", "missing file message");
  }
  // round trip of awkward doubles
  std::vector<std::tuple<int, int, double>> t{{0, 0, 0.1}, {0, 2, -1e-310}, {1, 1, 1.0 / 3.0}, {2, 0, 6.02214076e23},
                                              {2, 2, -0.0}};
  const CsrMatrixF m = from_triplets(3, t);
  save_matrix_market(p, m);
  const CsrMatrixF back = load_matrix_market(p);
  EXPECT(back.row_ptr == m.row_ptr && back.col_idx == m.col_idx, "round trip pattern");
  for (size_t k = 0; k < m.vals.size(); ++k)
    EXPECT(std::memcmp(&back.vals[k], &m.vals[k], sizeof(double)) == 0, "round trip bits");
  std::remove(p.c_str());
  std::printf("ok\n");
  return 0;
}
